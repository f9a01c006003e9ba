// Host-visible launch interfaces of the per-layer kernels (bb_layers.cu),
// attention (bb_attn.cu) and control kernels (bb_control.cu).
#pragma once
#include <cuda_runtime.h>

#include "bb_gemm.cuh"
#include "bb_state.cuh"

namespace bb {

struct Weights {
  const void* emb;    // [n_ext][d] T
  const void* pos;    // [max_len][d] T (arch 0)
  const void* wqkv;   // [layers][qkv_out][d] T
  const float* bqkv;  // [layers][qkv_out] or null
  const void* wo;     // [layers][d][attn_dim] T
  const void* wgu;    // [layers][2*dff][d] T, gate/up interleaved in 64-row blocks
  const void* wd;     // [layers][d][dff] T
  const float* ln1;   // [layers][d] (arch 1)
  const float* ln2;   // [layers][d]
  const float* lnf;   // [d]
  const void* head;   // [n_out][d] T
  const float* rope;  // [max_len][hd/2][2] (cos, sin), arch 1
};

struct PartRef {      // where a GEMM left its fp32 partial planes
  const float* part;
  long long plane;
  int ldp;
  SplitK sk;
};

// ---- per-layer kernels (templated on storage type inside) ----
cudaError_t launch_embed(const Dims& D, const Sess& S, const Pass& P, const Weights& W, cudaStream_t st);
cudaError_t launch_post_qkv(const Dims& D, const Sess& S, const Pass& P, const DevState& st, const Weights& W,
                            int layer, const PartRef& pr, cudaStream_t s);
cudaError_t launch_post_residual(const Dims& D, const Pass& P, const PartRef& pr, const float* ln, cudaStream_t s);
cudaError_t launch_post_gu(const Dims& D, const Pass& P, const PartRef& pr, cudaStream_t s);
// TMA views of the K / V page pools for the warp-specialized attention:
// [layers * R * pool * nkv * ps rows][hd] bf16, boxes of one 16-row page x 64 dims, 128-byte swizzle
struct AttnMaps {
  CUtensorMap k, v, kl, vl;  // kl / vl: the lo pools (bf16x2), else copies of k / v
  bool ok;
};
void attn_prepare();  // host-side occupancy queries (call outside stream capture)
// tflags: bb_session_desc.test_flags (tests only)
cudaError_t launch_attn(const Dims& D, const Sess& S, const Pass& P, const DevState& st, const AttnMaps& am, int layer,
                        int tflags, cudaStream_t s);
cudaError_t launch_attn_keys(const Dims& D, const Sess& S, const Pass& P, const DevState& st, cudaStream_t s);
cudaError_t launch_gather_head(const Dims& D, const Sess& S, const Pass& full, const Pass& blk, const Head& H,
                               int branch_filter, cudaStream_t s);
cudaError_t launch_head_logits(const Dims& D, const Pass& blk, const Head& H, float* logits, float* probs,
                               cudaStream_t s);
cudaError_t launch_head_tiles_f32(const Dims& D, const Pass& blk, const Head& H, cudaStream_t s);
cudaError_t launch_head_reduce(const Dims& D, const Sess& S, const Pass& blk, const Head& H, const DevState& st,
                               cudaStream_t s);

// ---- control kernels ----
cudaError_t launch_prefill_init(const Dims& D, const Sess& S, const DevState& st, const Pass& full, const Pass& blk,
                                const Head& H, cudaStream_t s);
cudaError_t launch_prefill_post(const Dims& D, const Sess& S, const DevState& st, const Pass& blk, const Head& H,
                                cudaStream_t s);
cudaError_t launch_block_bases(const Dims& D, const Sess& S, const DevState& st, const Pass& blk, const Head& H,
                               cudaStream_t s);
cudaError_t launch_block_pack(const Dims& D, const Sess& S, const DevState& st, const Pass& blk, const Head& H,
                              cudaStream_t s);
cudaError_t launch_copy_pages(const Dims& D, const Sess& S, const DevState& st, int with_pm, cudaStream_t s);
cudaError_t launch_step_commit(const Dims& D, const Sess& S, const DevState& st, const Pass& blk, const Head& H,
                               cudaStream_t s);
cudaError_t launch_merge_prep(const Dims& D, const Sess& S, const DevState& st, const Weights& W, cudaStream_t s);
cudaError_t launch_merge_sync(const Dims& D, const Sess& S, const DevState& st, int after_prefill, cudaStream_t s);
cudaError_t launch_refresh_begin(const Dims& D, const Sess& S, const DevState& st, const Pass& blk, const Head& H,
                                 cudaStream_t s);
cudaError_t launch_refresh_pack(const Dims& D, const Sess& S, const DevState& st, const Pass& full, const Pass& blk,
                                const Head& H, int branch, cudaStream_t s);
cudaError_t launch_refresh_end(const Dims& D, const Sess& S, const DevState& st, cudaStream_t s);
// KV-space diagnostics (log_kv / log_consistency)
cudaError_t launch_kv_scatter(const Dims& D, const Sess& S, const DevState& st, int r, int k, const float* src,
                              cudaStream_t s);
cudaError_t launch_seam_init(const Dims& D, const Sess& S, const DevState& st, cudaStream_t s);
cudaError_t launch_seam_block_pack(const Dims& D, const Sess& S, const DevState& st, const Pass& blk, const Head& H,
                                   int mask, int use_target, cudaStream_t s);
cudaError_t launch_seam_full_pack(const Dims& D, const Sess& S, const DevState& st, const Pass& full, const Pass& blk,
                                  const Head& H, int k, int use_target, cudaStream_t s);
cudaError_t launch_kv_gather(const Dims& D, const Sess& S, const DevState& st, int r, int k, float* dst,
                             cudaStream_t s);
cudaError_t launch_fresh_pack(const Dims& D, const Sess& S, const DevState& st, const Pass& full, int r, int k,
                              int* save, cudaStream_t s);
cudaError_t launch_fresh_restore(const Sess& S, const DevState& st, int r, int k, const int* save, cudaStream_t s);
cudaError_t launch_sqdiff_norm(const float* a, const float* b, long long n, double* part, int n_part, double* out,
                               cudaStream_t s);
// vanilla_decode (decoding.py:279-321): round = pack -> full pass -> head -> commit
cudaError_t launch_vanilla_pack(const Dims& D, const Sess& S, const DevState& st, const Pass& full, const Pass& blk,
                                const Head& H, cudaStream_t s);
cudaError_t launch_vanilla_commit(const Dims& D, const Sess& S, const DevState& st, const Pass& blk, const Head& H,
                                  cudaStream_t s);
cudaError_t launch_debug_commit(const float* probs, int n, int n_out, const int* pos, int* row, float tau, int* out,
                                int* count, cudaStream_t s);
cudaError_t launch_debug_merge(const Dims& D, const Sess& S, const DevState& st, const float* probmaps, int n_out,
                               cudaStream_t s);

}  // namespace bb
