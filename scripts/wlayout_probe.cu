// Weight-stream layout probe: how fast can 148 CTAs pull a [M][K] bf16 weight
// matrix through a TMA ring in stream-K order (no MMA)?
//   layout 0: row-major W[M][K], box {64 cols, 128 rows}: 128 rows x 128 B per box
//   layout 1: tile-packed W'[(mt*KB+kb)*128 + r][64]: the same box is 16 KB contiguous
//   layout 2: tile-packed, 1D cp.async.bulk of 16 KB (no swizzle; bandwidth only)
// 4 copies (4 x M x K x 2 B) rotate so nothing is L2-resident between launches.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2605_29233_b200/csrc
//        scripts/wlayout_probe.cu -o scripts/wlayout_probe -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "bb_common.cuh"
using namespace bb;

template <int ST>
__global__ void __launch_bounds__(64) k_stream(const __grid_constant__ CUtensorMap tm, const uint8_t* flat, int layout,
                                               int M, int K, unsigned long long* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * 16384);
  uint64_t* empty = full + ST;
  const int KB = K / 64, MT = M / 128;
  const long long T = (long long)MT * KB;
  const long long u0 = T * blockIdx.x / gridDim.x, u1 = T * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_first();
    int st = 0;
    uint32_t ph = 0;
    for (long long u = u0; u < u1; ++u) {
      const int mt = (int)(u / KB), kb = (int)(u % KB);
      mbar_wait(&empty[st], ph ^ 1);
      mbar_expect_tx(&full[st], 16384);
      if (layout == 0) {
        tma_load_2d(smem + st * 16384, &tm, &full[st], kb * 64, mt * 128, pol);
      } else if (layout == 1) {
        tma_load_2d(smem + st * 16384, &tm, &full[st], 0, (int)(u * 128), pol);
      } else {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                smem_u32(smem + st * 16384)),
            "l"(flat + u * 16384), "r"(16384), "r"(smem_u32(&full[st])), "l"(pol)
            : "memory");
      }
      if (++st == ST) {
        st = 0;
        ph ^= 1;
      }
    }
  } else if (threadIdx.x == 32) {
    int st = 0;
    uint32_t ph = 0;
    unsigned long long acc = 0;
    for (long long u = u0; u < u1; ++u) {
      mbar_wait(&full[st], ph);
      acc += *reinterpret_cast<volatile uint32_t*>(smem + st * 16384 + (u & 63) * 4);
      mbar_arrive(&empty[st]);
      if (++st == ST) {
        st = 0;
        ph ^= 1;
      }
    }
    if (acc == 0x123456789ull) *sink = acc;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;
static bool mk(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int ST>
static void run(int M, int K, int grid) {
  const size_t bytes = (size_t)M * K * 2;
  const int NC = 4;
  std::vector<uint8_t*> w(NC);
  for (int c = 0; c < NC; ++c) {
    cudaMalloc(&w[c], bytes);
    cudaMemset(w[c], c + 1, bytes);
  }
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int smem = ST * 16384 + 2048;
  cudaFuncSetAttribute(k_stream<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int layout = 0; layout < 3; ++layout) {
    std::vector<CUtensorMap> tm(NC);
    for (int c = 0; c < NC; ++c) {
      if (layout == 0) mk(&tm[c], w[c], K, M, 128);
      else mk(&tm[c], w[c], 64, (uint64_t)M * K / 64, 128);
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 8; ++i) k_stream<ST><<<grid, 64, smem>>>(tm[i % NC], w[i % NC], layout, M, K, sink);
    const int R = 40;
    cudaEventRecord(a);
    for (int i = 0; i < R; ++i) k_stream<ST><<<grid, 64, smem>>>(tm[i % NC], w[i % NC], layout, M, K, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1000.0 / R;
    printf("M=%5d K=%5d stages=%2d grid=%3d layout=%d (%s): %7.2f us/launch  %6.0f GB/s  [%s]\n", M, K, ST, grid,
           layout, layout == 0 ? "row-major 2D" : layout == 1 ? "tile-packed 2D" : "tile-packed 1D", us,
           bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  for (int c = 0; c < NC; ++c) cudaFree(w[c]);
  cudaFree(sink);
}

int main() {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int shapes[4][2] = {{12288, 4096}, {4096, 4096}, {24576, 4096}, {4096, 12288}};  // qkv, o, gate_up, down
  for (auto& s : shapes) {
    run<6>(s[0], s[1], sms);
    run<12>(s[0], s[1], sms);
  }
  run<6>(12288, 4096, 2 * sms);
  return 0;
}
