// GEMM interfaces shared by the launchers and the fused post-GEMM kernels.
//
// All projections are "weights-stationary, activations-streaming" TN GEMMs:
//   out[row][n] = sum_k X[row][k] * W[n][k]      (W: [n_out][K], X: [rows][K], both K-major)
// computed as D^T = W . X^T on tcgen05 (M = 128 weight rows per tile, N = BN
// activation rows), so a decode step with only ~56 window rows still issues
// full M=128 MMAs and every weight byte is read from HBM exactly once.
//
// Work is split stream-K over (tile, k-block): CTA c owns k-blocks
// [c*T/G, (c+1)*T/G) of the flattened (tile-major) space, tiles ordered
// chunk-outer (tile = chunk * n_ntiles + ntile) so that with several row
// chunks (full passes, batched sessions) CTAs c and c + G/n_chunks stream the
// same weight tiles at the same time: one HBM read, the other hits L2 and writes one fp32
// partial "plane" per tile piece.  The consumer kernel (post-QKV / post-O /
// ...) sums the pieces of a tile in slot order, so the reduction is
// deterministic and no fp32 atomics are used.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace bb {

struct SplitK {
  long long T;   // total k-blocks (= n_tiles * KB); 0 => single slot (SIMT path)
  int KB;        // k-blocks per tile
  int G;         // CTAs
  int n_chunks;  // row chunks per weight tile
  int n_ntiles;  // 128-row weight tiles; flattened tile = chunk * n_ntiles + ntile (chunk-outer)
  int BN;        // rows per chunk
  const unsigned char* ns_tab;  // optional [n_tiles] precomputed piece counts
  const int* rows_dyn;          // compacting sessions: device scalar of rows in use; the GEMM
                                // computes only ceil(rows/BN) chunks
  int np;                       // > 0: fixed pieces per tile (compacting sessions; ns = np)
};

// owner CTA of flattened k-block y (largest c with floor(c*T/G) <= y)
__host__ __device__ inline int sk_owner(long long y, long long T, int G) {
  return (int)(((y + 1) * (long long)G - 1) / T);
}
__host__ __device__ inline int sk_nslots(const SplitK& s, int row, int n) {
  if (s.T == 0) return 1;
  if (s.np > 0) return s.np;
  const long long tile = (long long)(row / s.BN) * s.n_ntiles + (n >> 7);
#ifdef __CUDA_ARCH__
  if (s.ns_tab != nullptr) return s.ns_tab[tile];
#endif
  const long long first = tile * s.KB, last = first + s.KB - 1;
  return sk_owner(last, s.T, s.G) - sk_owner(first, s.T, s.G) + 1;
}

// Sum of the partial planes for output element (row, n).
__device__ __forceinline__ float part_sum(const float* __restrict__ part, long long plane, int ldp,
                                          const SplitK& s, int row, int n) {
  const int ns = sk_nslots(s, row, n);
  const float* p = part + (long long)row * ldp + n;
  float acc = p[0];
  for (int i = 1; i < ns; ++i) acc += p[(long long)i * plane];
  return acc;
}

// Epilogue of a whole-tile (mode 1) GEMM: kind 1 = LM head + confidence.
struct EpiArgs {
  int kind;
};

struct GemmTcParams {
  // mode 0: stream-K into fp32 partial planes (consumed by post kernels)
  // mode 1: whole tiles round-robin over a persistent grid, epilogue from TMEM
  //         (epi.kind 1 = LM head)
  // mode 2: whole tiles round-robin into partial plane 0 (one piece per tile), tiles in
  //         groups of gc row chunks, weight-tile-major inside a group: a round's tiles
  //         share a few weight tiles and the group's activations stay in L2 (large
  //         full passes, where stream-K's spread-out ranges re-streamed every weight
  //         tile from HBM once per row chunk)
  int n_out, K, n_ntiles, n_chunks, KB, mode, gc;
  // bf16x2 activations: 0, or the real rows per chunk (= BN/2).  The B tile
  // then stacks the chunk's hi rows [0, half) and lo rows [half, BN) (two TMA
  // loads), the MMA runs N = BN, and the epilogue adds accumulator columns j
  // and half + j: out = W.(x_hi + x_lo) with fp32 accumulation
  int half;
  int rows_alloc;
  const int* rows_valid;  // device scalar or nullptr
  const int* rows_dyn;    // compacting sessions: rows in use (device scalar); only those chunks are computed
  int np;                 // mode 0: > 0 = fixed pieces per tile (see UnitIter)
  const int* skip;        // device scalar or nullptr: nonzero => no-op
  // mode 0
  float* part;
  long long plane;
  int ldp;
  // mode 1
  float4* head_part;  // [rows_alloc][n_ntiles] = (max, argmax bits, sumexp, 0)
  const float* boost;
  const int* tgt;
  float head_scale, spike_cut, spike_gain;
  float* raw_out;     // optional [rows_alloc][n_out]: raw dot products (materialised logits)
  // live per-launch timing (%globaltimer): this launch site's {min start, max end}
  unsigned long long* tstat;
  // timeline sessions, one GEMM kind (BB_GPH_KIND): per-CTA phase sums [CTAs,
  // resident before the wait, first stage landed, last MMA issued, first tile
  // stored, end] (ns, from the dependency wait's return; [1] before it)
  unsigned long long* ph;
  unsigned long long* klog;
  int klog_cap, klog_id;
  EpiArgs epi;
};

struct TcGemm {
  CUtensorMap tmA, tmB, tmB2;  // tmB2: lo plane of the activations (bf16x2), else unused
  const void* W;
  GemmTcParams p;
  SplitK sk;
  int BN, grid, max_slots;
};

// host API (bb_gemm.cu).  mode 0 = stream-K planes, 1 = LM head
// X_lo != nullptr: bf16x2 activations (BN real rows per chunk, MMA N = 2 BN)
bool tc_gemm_setup(TcGemm& g, const void* W, int n_out, int K, const void* X, int rows_alloc, int BN,
                   int mode, int max_grid, const void* X_lo = nullptr);
cudaError_t tc_gemm_launch(const TcGemm& g, cudaStream_t s);
// mode 0 -> mode 2 when the tiles fill at least `min_rounds` rounds of the grid
// (full passes; never for compacting sessions, whose consumers read np planes)
void tc_gemm_round_robin(TcGemm& g, int min_rounds, int act_row_bytes);
// 2-D bf16 tensor map [outer][inner], boxes of box_outer rows x 64 elements, 128-byte swizzle
bool tma_map_bf16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_outer);

struct SimtGemm {
  const float* W;
  const float* X;
  int n_out, K, rows_alloc;
  const int* rows_valid;
  const int* skip;
  float* out;
  int ldo;
};
cudaError_t simt_gemm_launch(const SimtGemm& g, cudaStream_t s);

}  // namespace bb
