// Kernel-level entry points used by the unit tests (exported C-ABI, see
// include/bb200.h "debug / unit-test entry points").
#include <stdio.h>
#include <string.h>

#include "bb_common.cuh"
#include "bb_launch.cuh"
#include "bb_gemm.cuh"
#include "bb200.h"

namespace bb {
__global__ void k_reduce_planes(const float* part, long long plane, int ldp, SplitK sk, int rows, int n_out,
                                float* out) {
  pdl_enter();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)rows * n_out) return;
  const int row = (int)(i / n_out), n = (int)(i % n_out);
  out[i] = part_sum(part, plane, ldp, sk, row, n);
}
}  // namespace bb

using namespace bb;

extern "C" {

// out[row][n] = sum_k X[row][k] W[n][k] via the tcgen05 stream-K kernel (mode 0)
// or the LM-head epilogue (mode 1: out = float4 [rows][ceil(n_out/128)]).
// `work` must hold max_slots * rows * n_out floats (mode 0); pass NULL to query
// the required float count in *work_floats.
BB_API int bb_debug_gemm_tc(const void* W, const void* X, void* out, int n_out, int K, int rows, int BN, int mode,
                     int max_grid, float* work, long long* work_floats, const int* tgt, const float* boost,
                     float head_scale, float spike_cut, float spike_gain, void* stream) {
  TcGemm g;
  if (!tc_gemm_setup(g, W, n_out, K, X, rows, BN, mode, max_grid)) return -3;
  const long long need = mode == 0 ? (long long)g.max_slots * rows * n_out : 0;
  if (work_floats) *work_floats = need;
  if (out == nullptr) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0) {
    g.p.part = work;
  } else {
    g.p.head_part = (float4*)out;
    g.p.tgt = tgt;
    g.p.boost = boost;
    g.p.head_scale = head_scale;
    g.p.spike_cut = spike_cut;
    g.p.spike_gain = spike_gain;
  }
  if (tc_gemm_launch(g, s) != cudaSuccess) return -10;
  if (mode == 0) {
    const long long n = (long long)rows * n_out;
    launch_k(k_reduce_planes, dim3((unsigned)((n + 255) / 256)), dim3(256), (size_t)(0), s, work, g.p.plane, g.p.ldp, g.sk, rows, n_out,
                                                                 (float*)out);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -10;
}

BB_API int bb_debug_gemm_simt(const float* W, const float* X, float* out, int n_out, int K, int rows, void* stream) {
  SimtGemm g{W, X, n_out, K, rows, nullptr, nullptr, out, n_out};
  return simt_gemm_launch(g, (cudaStream_t)stream) == cudaSuccess ? 0 : -10;
}
}

#include "bb_layers.cuh"

extern "C" {

// confidence_transition seam (decoding.py:108-129) on caller probabilities.
// probs [n][n_out] fp32, pos [n] (masked window positions, ascending), row [L]
// (mutated), out [n][2] (pos, tok) pairs, count [1].  All device pointers.
BB_API int bb_commit_probs(const float* probs, int n, int n_out, const int* pos, int* row, float tau, int* out,
                           int* count, void* stream) {
  if (n < 0 || n_out < 1) return BB_ERR_CONTRACT;
  if (n == 0) return cudaMemsetAsync(count, 0, 4, (cudaStream_t)stream) == cudaSuccess ? BB_OK : BB_ERR_CUDA;
  return launch_debug_commit(probs, n, n_out, pos, row, tau, out, count, (cudaStream_t)stream) == cudaSuccess
             ? BB_OK
             : BB_ERR_CUDA;
}

// merge_sync seam (scheduler.py:144-209) on caller state: rows [B][L] int32
// (mutated), branch [B][8] int32 (start,end,done,decoded,merged,block_size;
// mutated), covered [B][L] uint8 (mutated), probmaps [B][L][n_out] fp32,
// events [cap][20] int32 + ctrl [32] int32 (ctrl[C_NEV] = #events).
BB_API int bb_merge_sync_maps(int n_branches, int L, int prompt_len, int vocab_size, int* rows, int* branch,
                              unsigned char* covered, const float* probmaps, int n_out, float tau_merge,
                              float tau_sync, int merge_enabled, int sync_enabled, int* events, int ev_cap,
                              int* ctrl, float* ptab, unsigned char* ptab_ok, void* stream) {
  if (n_branches < 1 || n_branches > MAXB || L < 1) return BB_ERR_CONTRACT;
  Dims D;
  memset(&D, 0, sizeof(D));
  D.V = vocab_size;
  Sess S;
  memset(&S, 0, sizeof(S));
  S.R = 1;
  S.B = n_branches;
  S.L = L;
  S.P = prompt_len;
  S.G = L - prompt_len;
  S.tau_merge = tau_merge;
  S.tau_sync = tau_sync;
  S.merge_en = merge_enabled;
  S.sync_en = sync_enabled;
  S.trace = 1;
  S.ev_cap = ev_cap;
  DevState st;
  memset(&st, 0, sizeof(st));
  st.tokens = rows;
  st.br = branch;
  st.covered = covered;
  st.ctrl = ctrl;
  st.events = events;
  st.ptab = ptab;
  st.ptab_ok = ptab_ok;
  return launch_debug_merge(D, S, st, probmaps, n_out, (cudaStream_t)stream) == cudaSuccess ? BB_OK : BB_ERR_CUDA;
}
}
