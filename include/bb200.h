/* bb200.h — C-ABI of the B200-native BlockBatch batched denoising step.
 *
 * Plain C types only (pointers, sizes, ints, floats): no torch types.  Every
 * call returns int (0 = OK, negative = error code below) and takes the CUDA
 * stream to enqueue on as `void*` (a cudaStream_t).  Device buffers passed in
 * are caller-owned; handles are not thread-safe (one stream per session).
 *
 * The reference has no native code; its seams are Python functions.  Each
 * entry point below names the reference interface it replaces
 * (/root/reference/pkg/src/blockbatch/<file>:<line>).
 */
#ifndef BB200_H
#define BB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BB_API __attribute__((visibility("default")))

/* ---- error codes (mapped by the Python wrapper onto errors.py:4-17) ---- */
#define BB_OK 0
#define BB_ERR_CONFIG (-1)     /* ConfigError   (errors.py:4)  */
#define BB_ERR_CONTRACT (-2)   /* ContractError (errors.py:8)  */
#define BB_ERR_STATE (-3)      /* StateError    (errors.py:12) */
#define BB_ERR_RUNAWAY (-4)    /* RunawayError  (errors.py:16) */
#define BB_ERR_CUDA (-10)      /* CUDA launch / runtime failure */
#define BB_ERR_NOMEM (-11)     /* workspace too small           */

/* ---- model ------------------------------------------------------------- */
#define BB_ARCH_REF 0    /* reference synthetic denoiser (model.py:278-319): learned positions,
                            single head with head_dim = d_model, no norm, no MLP */
#define BB_ARCH_LLADA 1  /* LLaDA-8B / Dream-7B shape: RMSNorm, RoPE, MHA/GQA, SwiGLU, final norm */
#define BB_DTYPE_F32 0   /* fp32 verification mode (SIMT kernels)            */
#define BB_DTYPE_BF16 1  /* bf16 weights/activations/KV, fp32 accumulate (tcgen05) */
#define BB_DTYPE_BF16X2 2 /* bf16 weights; every activation, q/K/V and head input stored as a
                             bf16 hi + lo pair (x = hi + lo, ~2^-17 relative), both halves fed to the
                             tcgen05 MMAs (parity-grade bf16: hd 128 only) */

/* ModelParams (model.py:115-133) + ModelDims (model.py:66-70) + the LLaDA/Dream shape. */
typedef struct {
  int arch, vocab_size, layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, max_len, qkv_bias, dtype;
  float rope_theta, norm_eps, gamma;
  int radius;
  float head_scale, spike_cut, spike_gain;
} bb_model_desc;

/* Device pointers (caller-owned).  Matrices are (out, in) row-major in the
 * model dtype; norms/bias fp32.  wgu interleaves gate/up rows in blocks of 64
 * (rows [128t,128t+64) = gate features [64t,64t+64), next 64 = up). */
typedef struct {
  const void* emb;   /* [vocab+2][d]                  */
  const void* pos;   /* [max_len][d]      (arch REF)   */
  const void* wqkv;  /* [layers][(nh+2nkv)*hd][d]      */
  const float* bqkv; /* [layers][(nh+2nkv)*hd] or NULL */
  const void* wo;    /* [layers][d][nh*hd]             */
  const void* wgu;   /* [layers][2*d_ff][d]            */
  const void* wd;    /* [layers][d][d_ff]              */
  const float* ln1;  /* [layers][d]                    */
  const float* ln2;  /* [layers][d]                    */
  const float* lnf;  /* [d]                            */
  const void* head;  /* [vocab+1][d]                   */
} bb_weights;

/* Replaces build_model's product (model.py:210-241) as the forward's parameter set. */
BB_API int bb_model_create(const bb_model_desc* desc, const bb_weights* w, void** model);
BB_API int bb_model_destroy(void* model);

/* ---- session: R requests x B block-size branches ------------------------ */
/* SchedulerConfig (scheduler.py:32-63) + device layout knobs. */
typedef struct {
  int n_requests, n_branches;
  int block_sizes[8];
  int prompt_len, gen_len;
  float tau_conf, tau_merge, tau_sync;
  int refresh_interval, merge_enabled, sync_enabled;
  int page_size;       /* KV page positions (power of two <= 32, def. 16) */
  int pages_per_item;  /* attention split (pages per work item, def. 4)  */
  int trace;           /* record trace events (TraceEvent, decoding.py:61-75) */
  int event_capacity;  /* events per request                              */
  int diagnostics;     /* 1: reserve scratch KV pages for bb_fresh_kv (log_consistency) */
  int test_flags;      /* tests only (0 on the product path): bit 0 = mma.sync attention at
                          head_dim 128; bit 1 = the single-role tcgen05 attention (k_attn_tc)
                          instead of the warp-specialized one; bit 2 = the warp-specialized
                          attention on 64-row instead of 128-row tiles; bit 3 = no block-pass
                          compaction in batched sessions; bits 4-7 = forced cluster size;
                          bit 10 = full-pass GEMMs always stream-K (no grouped whole tiles);
                          bit 11 = refresh as one full pass per branch (no stacked pass) */
  int logits;          /* 1: the LM head also keeps raw logits (bb_head_logits; forward observers) */
  int seam;            /* 1: step-operator seam session (bb_seam_*): private pages per branch */
  int hard_cap;        /* > 0: override the forward cap 4*G*B+16 (scheduler.py:310; tests) */
} bb_session_desc;

#define BB_VIEW_TOKENS 0   /* int32 [R][B][L]      branch rows              */
#define BB_VIEW_TARGET 1   /* int32 [R][G]         planted targets (input)  */
#define BB_VIEW_PROMPT 2   /* int32 [R][P]         prompts (input)          */
#define BB_VIEW_CTRL 3     /* int32 [R][32]        status, NFE, counters    */
#define BB_VIEW_BRANCH 4   /* int32 [R][B][8]      window, done, progress   */
#define BB_VIEW_EVENTS 5   /* int32 [R][cap][20]   trace records            */
#define BB_VIEW_COVERED 6  /* uint8 [R][B][L]      prob_covered             */
#define BB_VIEW_PM_M 7     /* fp32  [R][B][L]      prob-map max logit       */
#define BB_VIEW_PM_S 8     /* fp32  [R][B][L]      prob-map sum-exp         */
#define BB_VIEW_PAGES 9    /* int32 [R][B][n_lp]   KV page tables           */
#define BB_VIEW_REFC 10    /* int32 [R][pool]      page refcounts           */
#define BB_VIEW_HEAD_MASKED 11 /* int32 [NR]     head slot reports a masked position */
#define BB_VIEW_HEAD_M 12  /* fp32  [NR]           max logit of the slot     */
#define BB_VIEW_HEAD_S 13  /* fp32  [NR]           sum exp(logit - max)      */
#define BB_VIEW_HEAD_ARG 14 /* int32 [NR]          argmax (lowest id)        */
#define BB_VIEW_SLOT_POS 15 /* int32 [NR]          position of the slot      */
#define BB_VIEW_SLOT_BR 16 /* int32 [NR]           branch of the slot        */
#define BB_VIEW_INIT_GEN 17 /* int32 [R][G]        initial generation row (input): token or -1 =
                               mask (single_branch_decode preset, decoding.py:194-212) */
#define BB_VIEW_COUNT 18

BB_API int bb_session_workspace_bytes(const void* model, const bb_session_desc* d, size_t* bytes);
BB_API int bb_session_create(void* model, const bb_session_desc* d, void* workspace, size_t bytes, void** sess);
BB_API int bb_session_destroy(void* sess);
BB_API int bb_session_view(const void* sess, int which, long long* offset, long long* bytes);
BB_API int bb_session_info(const void* sess, int* out, int n);
BB_API int bb_session_ctrl(void* sess, int* host_out, void* stream);

/* ---- the step ------------------------------------------------------------ */
/* init_full_forward + per-branch commit + advance + merge_sync (scheduler.py:80-89, 283-307) */
BB_API int bb_prefill(void* sess, void* stream);
/* one loop iteration without refresh: active set, pack, fused forward over all
 * active windows (1 NFE), Eq. 1 commit, EOS, advance, merge/sync
 * (scheduler.py:92-131, 322-372; decoding.py:108-191) */
BB_API int bb_block_step(void* sess, void* stream);
/* periodic refresh (scheduler.py:373-391) */
BB_API int bb_refresh(void* sess, void* stream);
/* block step (+ refresh), optionally replayed from a captured CUDA graph */
BB_API int bb_iteration(void* sess, int with_refresh, int use_graph, void* stream);
/* run_blockbatch (scheduler.py:225-394) for all requests of the session */
BB_API int bb_run(void* sess, int max_iterations, int use_graph, void* stream, int* iterations_out);
/* vanilla_decode (decoding.py:279-321) for all requests of a session that has
   one branch of block size gen_len: one full forward per round, tau 1.0.
   Replaces the reference's vanilla_decode (the baseline decoder of the
   paper's NFE comparison, test_acceptance.py:300-325). */
BB_API int bb_run_vanilla(void* sess, int max_iterations, int use_graph, void* stream, int* iterations_out);

/* ---- KV-space diagnostics (scheduler.py:268-281, 332-347, 376-390; the
   run_blockbatch log_kv / log_consistency modes).  The host runs the step in
   parts so the diagnostics see the caches between the forward and the
   commit/merge/sync that follows it. */
/* part 0: init + full forward + head; part 1: first commits, merge/sync, copies */
BB_API int bb_prefill_part(void* sess, int part, void* stream);
/* part 0: pack + copy-on-write copies (ctrl then holds the active set);
   part 1: forward + head; part 2: commit, EOS, merge/sync, copies */
BB_API int bb_block_step_part(void* sess, int part, void* stream);
/* kv_vectorize (model.py:346-352) of branch k of request r: fp32
   [layers][L][2][n_kv*head_dim] (keys before values) into dst (device) */
BB_API int bb_kv_gather(void* sess, int r, int k, float* dst, void* stream);
/* full_forward(row_k).cache vectorized the same way, without changing any
   session state (the pass writes into reserved scratch pages; needs
   diagnostics = 1 in the session desc) */
BB_API int bb_fresh_kv(void* sess, int r, int k, float* dst, void* stream);
/* ---- step-operator seams (model.py:322-343 full_forward / block_forward,
   scheduler.py:80-89 init_full_forward, :116-131 batched_block_forward) on a
   seam session (desc.seam = 1).  Rows, windows and targets are written through
   the TOKENS / BRANCH / TARGET views; caches through bb_kv_scatter. */
/* every branch of every request gets its own private pages (no aliasing) */
BB_API int bb_seam_init(void* sess, void* stream);
/* full = 0: block_forward of each branch in branch_mask over its window
   [start, end) and its current pages (the window's K/V rewritten in place);
   full = 1: full_forward of each branch in branch_mask (every position's K/V,
   head over every masked position; slot j of the branch = position j).
   use_target = 0: no agreement boost (target None, model.py:249-251). */
BB_API int bb_seam_forward(void* sess, int full, int branch_mask, int use_target, void* stream);
/* kv_vectorize inverse (model.py:346-352): fp32 [layers][L][2][kv_dim] (device)
   into branch k's pages of request r, rounded to the model dtype */
BB_API int bb_kv_scatter(void* sess, int r, int k, const float* src, void* stream);
/* DenoiseOutput of the last head pass (model.py:160-170): logits / probs fp32
   [head rows][n_out] (device; masked head slots written, others untouched).
   Needs desc.logits = 1 or desc.seam = 1. */
BB_API int bb_head_logits(void* sess, float* logits, float* probs, void* stream);
/* out[0] = ||a - b||_2 (b may be NULL), fp64 accumulation in a fixed order
   (partial sums in the session's workspace) */
BB_API int bb_sqdiff_norm(void* sess, const float* a, const float* b, long long n, double* out, void* stream);
BB_API int bb_version(void);
/* instrumentation: live per-launch GEMM timing and kernel-launch counters */
BB_API int bb_session_gemm_stats(void* sess, unsigned long long* host_out, int reset, void* stream);
/* Timeline sessions (BB_KLOG=1): phase offsets of the fused-QKV block
 * attention, out[8] = (CTAs, then summed ns from the PDL release to: rows and
 * keys loaded, phase-A loads issued, splice stored, cluster barrier passed,
 * chunk 0 landed, chunk loop done, end).  Averages = out[i] / out[0].
 * out[8..15]: one GEMM kind's phases (env BB_GPH_KIND = 8*full + kind, kind 0-3
 * = QKV, O, gate/up, down; default 1): (CTAs, summed ns resident before the
 * dependency wait, then from it to: first stage landed, last MMA issued, first
 * tile stored, end).  out must hold 16 values. */
BB_API int bb_session_phase_stats(void* sess, unsigned long long* out, int reset, void* stream);
BB_API int bb_session_counters(void* sess, long long* out);
BB_API int bb_session_klog(void* sess, unsigned long long* host_out, int cap, int reset, long long* n, void* stream);

/* ---- debug / unit-test entry points (kernel-level) --------------------- */
BB_API int bb_debug_gemm_tc(const void* W, const void* X, void* out, int n_out, int K, int rows, int BN, int mode,
                            int max_grid, float* work, long long* work_floats, const int* tgt, const float* boost,
                            float head_scale, float spike_cut, float spike_gain, void* stream);
BB_API int bb_debug_gemm_simt(const float* W, const float* X, float* out, int n_out, int K, int rows,
                              void* stream);

/* step-operator seams on caller-supplied state (bit-exact given identical
 * confidences; the same device code the fused step runs) */
BB_API int bb_commit_probs(const float* probs, int n, int n_out, const int* pos, int* row, float tau, int* out,
                           int* count, void* stream);
BB_API int bb_merge_sync_maps(int n_branches, int L, int prompt_len, int vocab_size, int* rows, int* branch,
                              unsigned char* covered, const float* probmaps, int n_out, float tau_merge,
                              float tau_sync, int merge_enabled, int sync_enabled, int* events, int ev_cap,
                              int* ctrl, float* ptab, unsigned char* ptab_ok, void* stream);
/* device random-init (oracle/bb_oracle.py:hash_uniform); mode 1 = gate/up interleave */
BB_API int bb_fill_hash_uniform(void* dst, int dtype, long long n, unsigned long long seed, int tensor_id, float c,
                                long long start, int mode, int d, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BB200_H */
