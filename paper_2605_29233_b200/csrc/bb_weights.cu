// Device-side random-init of LLaDA/Dream-shape weights from a counter-based
// hash, bit-identical to oracle/bb_oracle.py:hash_uniform.  8B parameters are
// generated in place in a few ms instead of streaming 16 GB from the host.
#include "bb200.h"
#include "bb_common.cuh"

namespace bb {

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// u in (-1,1): ((h >> 41) - 2^22 + 0.5) / 2^22, then * c, each rounded once in fp32.
__device__ __forceinline__ float hash_value(uint64_t base, uint64_t idx, float c) {
  const uint64_t h = splitmix(idx + base);
  const int k = (int)(h >> 41) - (1 << 22);
  const float u = __fmul_rn(__fadd_rn((float)k, 0.5f), 1.0f / 4194304.0f);
  return __fmul_rn(u, c);
}

template <typename T>
__global__ void k_fill_hash(T* dst, long long n, uint64_t base_a, uint64_t base_b, float c, long long start, int mode,
                            int d) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    float v;
    if (mode == 0) {
      v = hash_value(base_a, (uint64_t)(start + e), c);
    } else {  // gate/up interleave in 64-row blocks
      const long long R = e / d, col = e % d;
      const long long t = R >> 7, w = R & 127;
      const long long f = 64 * t + (w < 64 ? w : w - 64);
      v = hash_value(w < 64 ? base_a : base_b, (uint64_t)(f * d + col), c);
    }
    stf(dst + e, v);
  }
}

}  // namespace bb

using namespace bb;

extern "C" BB_API int bb_fill_hash_uniform(void* dst, int dtype, long long n, unsigned long long seed, int tensor_id,
                                           float c, long long start, int mode, int d, void* stream) {
  if (!dst || n < 0 || (mode == 1 && d <= 0)) return BB_ERR_CONTRACT;
  const uint64_t ka = seed * 0x9E3779B97F4A7C15ull + (uint64_t)tensor_id * 0xD1B54A32D192ED03ull;
  const uint64_t kb = seed * 0x9E3779B97F4A7C15ull + (uint64_t)(tensor_id + 1) * 0xD1B54A32D192ED03ull;
  const long long blocks = (n + 255) / 256;
  const int grid = (int)(blocks < 4 * 148 * 8 ? (blocks > 0 ? blocks : 1) : 4 * 148 * 8);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == BB_DTYPE_BF16)
    k_fill_hash<__nv_bfloat16><<<grid, 256, 0, s>>>((__nv_bfloat16*)dst, n, ka, kb, c, start, mode, d);
  else
    k_fill_hash<float><<<grid, 256, 0, s>>>((float*)dst, n, ka, kb, c, start, mode, d);
  return cudaGetLastError() == cudaSuccess ? BB_OK : BB_ERR_CUDA;
}
