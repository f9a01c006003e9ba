// Probe of the tcgen05 conventions the tensor-core attention relies on
// (standalone: nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2605_29233_b200/csrc
// scripts/tc_probe.cu -o tc_probe -lcuda).  One CTA runs
//   mode 0: D[64 x N] = A[64 x 64] . B[N x 64]^T   (A, B K-major, SW128)
//   mode 1: D[64 x N] = A[64 x 64] . B[64 x N]      (B MN-major, SW128, two 64-wide MN atoms)
// with A[m][0] = m, A[m][1] = 64, B(k=0, n) = 1, B(k=1, n) = n, so D[m][n] = m + 64 n,
// dumps all 128 TMEM lanes x N/2.. columns and prints where each (m, n) landed.
#include <cstdio>
#include <cuda_bf16.h>
#include <cstdint>
#include "bb_common.cuh"

using namespace bb;

__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

template <int N>
__global__ void probe(int mode, float* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;             // [64][64] K-major
  uint8_t* sB = sm + 8192;      // mode 0: [N][64] K-major; mode 1: 2 x [64 k][64 n] MN-major
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  // zero
  for (int i = t; i < (8192 + 2 * 8192) / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  auto put = [&](uint8_t* base, int r, int k, float v) {  // element (row r, col k) of a [rows][64] SW128 tile
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(base + swz(r, k >> 3)) + (k & 7);
    *p = __float2bfloat16(v);
  };
  if (t < 64) {
    put(sA, t, 0, (float)t);
    put(sA, t, 1, 64.0f);
  }
  if (mode == 0) {
    for (int n = t; n < N; n += blockDim.x) {
      put(sB, n, 0, 1.0f);
      put(sB, n, 1, (float)n);
    }
  } else {
    // MN-major: atom a holds n in [64a, 64a+64); row = k
    for (int n = t; n < N; n += blockDim.x) {
      put(sB + (n >> 6) * 8192, 0, n & 63, 1.0f);
      put(sB + (n >> 6) * 8192, 1, n & 63, (float)n);
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (t < 32) tmem_alloc(&tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (t == 0) {
    uint32_t idesc = idesc_bf16_f32(64, N) | (mode == 1 ? (1u << 16) : 0u);
    for (int ks = 0; ks < 4; ++ks) {
      const uint64_t ad = sdesc_sw128(smem_u32(sA) + ks * 32);
      const uint64_t bd = mode == 0 ? sdesc_sw128(smem_u32(sB) + ks * 32) : desc_mn(smem_u32(sB) + ks * 2048, 8192, 1024);
      tc_mma_bf16(tb, ad, bd, idesc, ks > 0 ? 1u : 0u);
    }
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = t >> 5;
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tmem_ld32(tb + ((uint32_t)(32 * w) << 16) + c0, v);
    for (int c = 0; c < 32; ++c) out[(32 * w + (t & 31)) * N + c0 + c] = v[c];
  }
  tc_fence_before();
  __syncthreads();
  if (t < 32) {
    tc_fence_after();
    tmem_dealloc(tb, 256);
  }
}

template <int N>
static void run(int mode) {
  float* d;
  cudaMalloc(&d, 128 * N * 4);
  cudaMemset(d, 0xff, 128 * N * 4);
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<N><<<1, 128, 48 * 1024>>>(mode, d);
  cudaError_t e = cudaDeviceSynchronize();
  float* h = new float[128 * N];
  cudaMemcpy(h, d, 128 * N * 4, cudaMemcpyDeviceToHost);
  printf("mode %d N %d: %s\n", mode, N, cudaGetErrorString(e));
  // where did (m, n) land?  print per lane the first columns' decoded (m, n)
  int ok_interleaved = 0, ok_total = 0;
  for (int lane = 0; lane < 128; ++lane) {
    for (int c = 0; c < N; ++c) {
      const float v = h[lane * N + c];
      // expected under the "lanes 64+ hold the right half" layout
      if (c < N / 2) {
        const int m = lane & 63, n = c + (lane >= 64 ? N / 2 : 0);
        ++ok_total;
        if (v == (float)(m + 64 * n)) ++ok_interleaved;
      }
    }
  }
  printf("  interleaved-layout matches: %d / %d\n", ok_interleaved, ok_total);
  for (int lane : {0, 1, 15, 16, 31, 32, 47, 63, 64, 65, 96, 127}) {
    printf("  lane %3d:", lane);
    for (int c : {0, 1, 2, N / 2 - 1, N / 2, N - 1}) {
      const float v = h[lane * N + c];
      if (v != v) printf("  c%d=nan", c);
      else printf("  c%d=(m%d,n%d)%s", c, ((int)v) % 64, ((int)v) / 64, v == (float)(int)v ? "" : "~");
    }
    printf("\n");
  }
  delete[] h;
  cudaFree(d);
}

int main() {
  run<64>(0);
  run<128>(0);
  run<64>(1);
  run<128>(1);
  return 0;
}
