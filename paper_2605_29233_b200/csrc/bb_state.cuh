// Device-resident state of a BlockBatch session (a group of R requests, each
// with B block-size branches) and of its two forward passes.
//
// The whole Alg. 1 step runs on the device: the host enqueues a fixed kernel
// sequence per iteration (CUDA-graph capturable) and only polls a status word.
//
// HBM layout (request-major):
//   tokens  [R][B][L] int32          branch rows (SequenceRow.tokens, model.py:92-112)
//   br      [R][B][B_WORDS] int32    BranchState window/done/progress (decoding.py:78-93)
//   ctrl    [R][C_WORDS] int32       NFE counters, iteration, status, event count ...
//   prob map (BranchState.prob_map, decoding.py:88): per (r, b, pos) the head
//            input row h (T, d) + max logit m + sum-exp s + target boost, so
//            P_b(pos, v) = exp(logit(h, v) - m) / s is recomputed on demand
//            instead of storing L x n_out probabilities.
//   KV pages [layers][R*pool][n_kv][page][head_dim] (T) addressed through a
//            per-branch page table with refcounts: branches alias shared pages
//            (prefill prefix, sync) and copy-on-write before writing.
#pragma once
#include <stdint.h>

namespace bb {

constexpr int MAXB = 8;     // max branches per request
constexpr int EVW = 20;     // int32 words per trace event record
constexpr int ITW = 4;      // int32 words per attention item (mask, lp0, lp1, rep)
constexpr int QT = 32;      // query rows per attention CTA

enum EvKind {
  EV_INIT = 0, EV_BLOCK = 1, EV_DECODE = 2, EV_MERGE = 3, EV_SYNC = 4,
  EV_REFRESH = 5, EV_EOS_PENDING = 6, EV_EOS_READY = 7, EV_FINISH = 8
};
// event record: [kind, branch(-1=None), nfe0, nfe1, nfe2, a0, a1, a2, a3, prob_bits, decoded[MAXB], pad, pad]
enum EvField { E_KIND = 0, E_BRANCH, E_NFE0, E_NFE1, E_NFE2, E_A0, E_A1, E_A2, E_A3, E_PROB, E_DEC };

enum Ctrl {
  C_STATUS = 0,     // 0 running, 1 finished, <0 error code
  C_WINNER, C_EOS, C_ITER, C_SINCE_REFRESH, C_NFE0, C_NFE1, C_NFE2, C_NEV, C_REFRESH_DUE,
  C_EV_OVERFLOW, C_ACTIVE_MASK, C_REFRESH_MASK, C_NCOPY, C_NPMCOPY, C_MERGES, C_SYNCS,
  C_COMMITS, C_REFRESHES, C_BLOCK_ROWS, C_COW_PAGES, C_SHARED_PAGES, C_LAST_ACTIVE,
  C_WORDS = 32
};
enum Br { B_START = 0, B_END, B_DONE, B_DEC, B_MERGED, B_SIZE, B_WORDS = 8 };

struct Dims {
  int arch;  // 0 = reference synthetic denoiser, 1 = LLaDA/Dream shape
  int V, n_out, n_ext, layers, d, nh, nkv, hd, dff, max_len, qkv_bias, dtype;
  int split;  // BB_DTYPE_BF16X2: dtype 1 storage with a bf16 lo plane beside every bf16 activation
  int qkv_out, attn_dim, kv_dim, n_vtiles;
  float eps, gamma, head_scale, spike_cut, spike_gain, attn_scale;
  int radius;
  unsigned long long* klog;  // kernel timeline log ([0] count, then (id, t_ns) pairs) or null
  int klog_cap;
};

struct Sess {
  int R, B, P, G, L;
  int bs[MAXB];
  int off[MAXB];      // block-pass slot offset of branch k inside a request
  int NRq;            // block-pass rows per request
  int NR;             // block-pass rows (R * NRq)
  int NF;             // full-pass rows (R * L)
  float tau_conf, tau_merge, tau_sync;
  int refresh_interval, merge_en, sync_en;
  int ps, n_pp, n_gp, n_lp, pool;
  int ps_shift;       // log2(ps) (page sizes are powers of two)
  int ch_block;       // logical pages per attention item in block passes
  int max_items;      // attention items per request per pass
  int ev_cap, trace, hard_cap, max_copies;
  int diag;           // diagnostics session: the last n_lp pages of each request's pool are scratch
  int n_sms;          // SMs of the device (grid sizing)
  int compact;        // batched tcgen05 sessions: block-pass rows of the live requests only
                      // (Pass::req_base / rows_live), so finished requests cost no GEMM rows
};

struct DevState {
  int* tokens;
  int* target;  // [R][G]
  int* prompt;  // [R][P]
  int* init_gen;  // [R][G] initial generation row: token, or -1 = mask (presets)
  int* ctrl;
  int* br;
  uint8_t* covered;   // [R][B][L]
  void* pm_h;         // [R][B][L][d] T
  float* pm_m;        // [R][B][L]
  float* pm_s;
  float* pm_boost;
  int* pt;            // [R][B][n_lp]
  int* refc;          // [R][pool]
  int* freel;         // [R][pool]
  int* free_top;      // [R]
  int* copies;        // [R][max_copies][2]
  int* pm_copies;     // [R][MAXB][2]
  int* events;        // [R][ev_cap][EVW]
  float* ptab;        // [R][B][L][B] merge probability table
  uint8_t* ptab_ok;   // [R][B][L]
  void* kv_k;         // [layers][R*pool][nkv][ps][hd] T
  void* kv_v;
  long long kv_lo;    // split: element offset of the lo pool (kv_k + kv_lo, kv_v + kv_lo); 0 otherwise
  void* pm_h_lo;      // split: lo plane of pm_h (else null)
};

struct Pass {
  int rows_alloc;
  int full;           // 1 = full forward (prefill/refresh), 0 = block step
  int nseq = 1;       // full pass: sequences per request, L rows each -- 1 (prefill, per-branch
                      // passes), or B for the stacked refresh (request r, branch k at rows
                      // (r * B + k) * L); the attention's row groups are (request, sequence)
  int* slot_pos;      // [rows_alloc] (-1 = padding)
  int* slot_req;
  int* slot_br;
  int* slot_tok;
  long long* slot_kvoff;  // [rows_alloc] KV element offset of the row's (page, slot) within a layer
  int* rng_off;       // [R][MAXB] slot range of (request, branch)
  int* rng_cnt;
  int* items;         // [R][max_items][ITW]
  int* n_items;       // [R]
  int* skip;          // device flag (1 = pass is a no-op)
  int item_rows;      // row capacity per item in apart
  float* x;           // [rows_alloc][d] fp32 residual stream
  void* xn;           // [rows_alloc][d] T  (GEMM input)
  void* q;            // [rows_alloc][attn_dim] T
  void* attn;         // [rows_alloc][attn_dim] T
  void* act;          // [rows_alloc][dff] T
  // split (bf16x2) sessions: the lo planes of xn / q / attn / act (same shapes), else null
  void* xn_lo;
  void* q_lo;
  void* attn_lo;
  void* act_lo;
  float* apart;       // [R][max_items][item_rows][nh][hd+2]
  float* row_rope;    // [rows_alloc][hd/2][2] RoPE (cos, sin) of each row's position (block pass, arch 1) or null
  // key lists of the tensor-core attention, built once per pass (the page
  // tables do not change between layers): per (request, key tile) the keys
  // in lp-major order as (page_global * ps + row_in_page, branch mask)
  int* akeys;         // [R][n_kz][akey_cap][2]
  int* akey_n;        // [R][n_kz][2] (n_keys, first key of the generation pages)
  int akey_cap;
  int n_kz;           // key tiles per request (block pass: (1 << kz_shift)-row tiles; full pass: 1)
  int kz_shift;       // log2 rows per key tile: 7 for the M = 128 attention, else 6 (a key list of a
                      // 128-row tile serves its 64-row halves too: a superset of their keys)
  unsigned long long* atstat;  // live attention timing: [0..7] duration, [8..15] CTA start spread
  // block pass of a compacting session: per request the first slot of its NRq
  // slots this iteration (-1: finished), and the slots in use (a device
  // scalar the GEMMs size their work by); static r * NRq otherwise
  int* req_base;      // [R]
  int* rows_live;
  // L2 prefetch of the next GEMM's weights issued by the attention CTAs (HBM is
  // idle during the attention): layer l's bytes at pf_base + l * pf_layer_bytes
  const char* pf_base;
  long long pf_layer_bytes;
};

// Head (LM head + confidence) works on block-pass slots.
struct Head {
  int* masked;        // [rows] 1 = report this slot (masked window position)
  float* boost;       // [rows]
  int* tgt;           // [rows]
  float4* hpart;      // [rows][n_vtiles]
  float* logits;      // fp32 mode: [rows][n_out] raw dot products
  float* raw;         // bf16 mode, logits sessions: [rows][n_out] raw dot products (else null)
  float* res_conf;    // [rows]
  int* res_arg;
  float* res_m;
  float* res_s;
  int* skip;
};

// the segment-masked tensor-core attention derives its work from the page
// tables; only the SIMT (fp32 / head_dim 32,256) path needs planned items
__host__ __device__ inline bool uses_items(const Dims& D) {
  return !(D.dtype == 1 && (D.hd == 64 || D.hd == 128));
}

// row groups of a pass: one per request (block pass) or per (request, sequence) (full pass)
__host__ __device__ inline int pass_groups(const Sess& S, const Pass& P) { return P.full ? S.R * P.nseq : S.R; }

// first block-pass slot of request r (-1: finished, compacting sessions only)
__host__ __device__ inline int blk_base(const Sess& S, const Pass& blk, int r) {
#ifdef __CUDA_ARCH__
  if (S.compact) return blk.req_base[r];
#endif
  return r * S.NRq;
}

__host__ __device__ inline int lp_start(const Sess& s, int lp) {
  return lp < s.n_pp ? lp * s.ps : s.P + (lp - s.n_pp) * s.ps;
}
__host__ __device__ inline int lp_end(const Sess& s, int lp) {
  const int e = lp < s.n_pp ? (lp + 1) * s.ps : s.P + (lp - s.n_pp + 1) * s.ps;
  const int cap = lp < s.n_pp ? s.P : s.L;
  return e < cap ? e : cap;
}
__host__ __device__ inline int lp_of(const Sess& s, int pos) {
  return pos < s.P ? pos / s.ps : s.n_pp + (pos - s.P) / s.ps;
}

}  // namespace bb
