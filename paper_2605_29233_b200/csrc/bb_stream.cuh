// Layer-stream kernel (LSK): one persistent launch per layer of the block
// pass that runs the layer's projection GEMMs and their consumer ops as
// phases separated by grid-wide barriers, so the weight stream never stops at
// a kernel boundary:
//
//   attention(l) -> LSK(l) = [O -> residual+RMSNorm] [gate/up -> SwiGLU]
//                            [down -> residual+RMSNorm] [QKV(l+1) -> bias,RoPE,KV splice]
//
// (model.py:291-303 per layer, LLaDA/Dream shape).  The weight (A operand)
// producer has no data dependency, so it runs ahead through the phase
// boundaries and fills the shared-memory ring with the next GEMM's weights
// while the consumer op and the barrier of the previous phase are in flight;
// only the activation (B operand) loads wait for the barrier.  The ring is
// sized so the attention kernel of the next layer (launched early through
// PDL) can be resident next to it.
#pragma once
#include <cuda.h>

#include "bb_gemm.cuh"
#include "bb_layers.cuh"

namespace bb {

constexpr int LSK_MAXG = 4;
constexpr int LSK_BAR_WORDS = 3 * LSK_MAXG + 1;

enum LskPost { LSK_POST_NONE = 0, LSK_POST_RESIDUAL = 1, LSK_POST_SWIGLU = 2, LSK_POST_QKV = 3 };

struct LskGemm {
  int n_out, K, n_ntiles, n_chunks, KB, G;  // G = CTAs that own k-blocks (stream-K split, <= grid)
  long long T;                              // n_ntiles * n_chunks * KB
  long long plane;                          // elements per partial plane (rows_alloc * n_out)
  int max_ns;                               // largest stream-K piece count of a tile
  SplitK sk;                                // piece counts for the consumer op
  int post;                                 // LskPost
  const float* ln;                          // residual: RMSNorm gain of the next GEMM input (null = copy)
  const float* bias;                        // qkv: bias or null
  int layer;                                // qkv: KV layer written by the splice
  unsigned long long* tstat;                // live span of this GEMM phase or null
};

// everything but the tensor maps; copied to shared memory at kernel start so
// the consumer ops read it from smem (a reference to the kernel parameter
// itself would make the compiler build a per-thread local copy)
struct LskCore {
  LskGemm g[LSK_MAXG];
  int n_gemm;
  int flags;  // BB_LSK_FLAGS bit 0 (diagnostic): the weight producer waits at phase boundaries
  int rows;  // rows the consumer ops visit (block pass: R * NRq; the rest are padding)
  Dims D;
  Sess S;
  Pass P;
  DevState st;
  float* part;  // stream-K partial planes (shared by all phases)
  float* ss;    // [rows_alloc][d/128] residual sum-of-squares partials
  const float* rope;
  unsigned int* bar;          // [LSK_BAR_WORDS] self-resetting grid-barrier counters
  unsigned long long* tstat;  // whole-kernel live span or null
  unsigned long long* prof;   // CTA-0 phase profile [64] (BB_KLOG sessions) or null
};

struct LskParams {
  CUtensorMap tmA[LSK_MAXG];  // weights [n_out][K]
  CUtensorMap tmB[LSK_MAXG];  // activations [rows_alloc][K]
  LskCore c;
};

// host
int lsk_stages();
size_t lsk_smem(int stages);
bool lsk_add_gemm(LskParams& p, const TcGemm& g, int post, const float* ln, const float* bias, int layer,
                  unsigned long long* tstat);
cudaError_t lsk_launch(const LskParams& p, int grid, cudaStream_t s);

}  // namespace bb
