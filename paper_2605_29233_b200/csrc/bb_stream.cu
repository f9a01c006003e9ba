// Layer-stream kernel (see bb_stream.cuh).
//
// CTA layout (224 threads, exactly one CTA per SM, grid = #SMs):
//   warp 0 lane 0 : weight producer   TMA 128x64 W tiles of every phase, back to back
//   warp 1 lane 0 : MMA issuer        4 x tcgen05.mma M128 N=BN K16 per k-block
//   warps 2-5     : epilogue (TMEM -> fp32 partial planes) and the consumer ops
//   warp 6 lane 0 : activation producer  TMA BNx64 X tiles, after the phase barrier
// The ring stage's `full` barrier takes one arrival from each producer.
//
// Phase protocol (counters bar[] in global memory, one per event):
//   bar[3i]   : CTAs whose epilogue wrote all partial planes of GEMM i
//   bar[3i+1] : CTAs that finished step 1 of GEMM i's consumer op
//   bar[3i+2] : CTAs that finished step 2 (residual: the RMSNorm)
//   GEMM i+1's activation loads wait for the last of these its input needs;
//   each consumer step waits for the previous counter == grid.  The last CTA
//   to leave resets them.
// Every wait is bounded (trap instead of a hung GPU).
#include "bb_common.cuh"
#include "bb_launch.cuh"
#include "bb_stream.cuh"

namespace bb {

template <int BN, int STAGES>
struct LskCfg {
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr uint32_t TCOLS = 2 * BN <= 128 ? 128 : 256;
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * (A_BYTES + B_BYTES) + (2 * STAGES + 4) * 8 + 64;
};

// Poll with relaxed loads and acquire once: ld.acquire.gpu (and every gpu-scope
// fence) invalidates the SM's whole L1 (CCTL.IVALL), so an acquire per poll
// iteration would wipe the L1 lines and register spills of the other warps on
// the SM for as long as the wait lasts.
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_wait(const unsigned* p, unsigned target) {
  if (ld_relaxed_u32(p) < target) {
    const long long t0 = clock64();
    while (ld_relaxed_u32(p) < target) {
      __nanosleep(16);
      if (clock64() - t0 > 20000000000LL) __trap();
    }
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
// release-add without a returned value (no full fence, no L1 invalidation)
__device__ __forceinline__ void grid_arrive(unsigned* p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void lsk_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// live span of a phase: min start / max end over CTAs; the last CTA folds it
__device__ __forceinline__ void span_begin(unsigned long long* ts) {
  if (ts != nullptr) atomicMin(&ts[0], globaltimer_ns());
}
__device__ __forceinline__ void span_end(unsigned long long* ts, unsigned n) {
  if (ts == nullptr) return;  // (timing only: no fences, see grid_wait)
  atomicMax(&ts[1], globaltimer_ns());
  if (atomicAdd(&ts[2], 1ull) == n - 1) {
    const unsigned long long t0 = atomicAdd(&ts[0], 0ull), t1 = atomicAdd(&ts[1], 0ull);
    atomicAdd(&ts[3], t1 - t0);
    atomicAdd(&ts[4], 1ull);
    atomicExch(&ts[0], ~0ull);
    atomicExch(&ts[1], 0ull);
    atomicExch(&ts[2], 0ull);
  }
}

// CTA-0 phase profile (BB_KLOG sessions): prof[k] += t(event k) - t(release)
__device__ __forceinline__ void lsk_prof(unsigned long long* prof, int k, unsigned long long t0) {
  if (prof != nullptr && blockIdx.x == 0) atomicAdd(&prof[k], globaltimer_ns() - t0);
}

// stream-K range of CTA c in GEMM g, walked as (tile, kb0, kb1, slot) units
struct LskUnits {
  long long x, end;
  int KB, c, G;
  long long T;
  __device__ LskUnits(const LskGemm& g, int c_) : KB(g.KB), c(c_), G(g.G), T(g.T) {
    if (c < G) {
      x = (long long)c * T / G;
      end = (long long)(c + 1) * T / G;
    } else {
      x = end = 0;
    }
  }
  __device__ bool next(int& tile, int& kb0, int& kb1, int& slot) {
    if (x >= end) return false;
    tile = (int)(x / KB);
    kb0 = (int)(x % KB);
    const long long rem = end - x;
    kb1 = (int)((long long)kb0 + rem < KB ? kb0 + rem : KB);
    slot = c - sk_owner((long long)tile * KB, T, G);
    x += kb1 - kb0;
    return true;
  }
  __device__ long long count() const { return end - x; }
};

constexpr int LSK_POST_THREADS = 256;  // warps 7-14: consumer ops
#ifndef LSK_RB_RES
#define LSK_RB_RES 1
#endif
#ifndef LSK_RB_SW
#define LSK_RB_SW 2
#endif
#ifndef LSK_NS_RES
#define LSK_NS_RES 8
#endif
#ifndef LSK_NS_SW
#define LSK_NS_SW 2
#endif
#ifndef LSK_NS_QKV
#define LSK_NS_QKV 4
#endif
// ---------------------------------------------------------------- consumer ops
// Same math as k_post_residual / k_post_gu / k_post_qkv (bb_layers.cu), spread
// over the grid's 148 x 4 epilogue warps.  The partial planes were written by
// other SMs inside this launch: L2-only loads (ld.cg), and every thread issues
// all loads of U work items (NS planes each, predicated) before it sums them,
// so a phase costs a couple of L2 round trips instead of a dependent chain.
// Planes are summed in slot order, as in the separate kernels (deterministic).
using bf16 = __nv_bfloat16;

// plain (weak) loads: the phase barrier's acquire (thread 0's fence after the
// counter load, then bar.sync) orders them after the producers' writes; ld.cg
// compiles to STRONG.GPU loads here, which are much slower
__device__ __forceinline__ float4 ldcg4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float ldcg1(const float* p) { return *p; }
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void add4(float4& a, const float4& b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}
__device__ __forceinline__ void st_bf16x4(bf16* p, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = u;
}

// Thread mapping of every op: thread t of the grid owns column vector
// cv = t % ncv (4 consecutive output columns) and visits rows rg, rg + nrg, ...
// (rg = t / ncv, nrg = grid threads / ncv): all column math is hoisted out of
// the row loop, and consecutive lanes of a warp own consecutive columns of the
// same row (coalesced; for the residual a warp is exactly one 128-column
// segment, so a warp sum is that segment's sum of squares).
struct ColMap {
  int cv, rg, nrg;
  __device__ ColMap(int ncv, int et) {
    const int t = blockIdx.x * LSK_POST_THREADS + et, nthr = gridDim.x * LSK_POST_THREADS;
    cv = t % ncv;
    rg = t / ncv;
    nrg = nthr / ncv;
  }
};
// stream-K piece count of (row, column c) for BN = 64 row chunks
__device__ __forceinline__ int lsk_ns(const LskGemm& g, int row, int c) {
  return g.sk.ns_tab[(row >> 6) * g.n_ntiles + (c >> 7)];
}

// Each thread processes its rows in batches of RB: every load of the batch is
// issued before the first store (stores could alias later loads, so the
// compiler would otherwise serialise one L2 round trip chain per row).

// residual, step 1: x += sum(planes); per (row, 128-column segment) sum of squares -> ss
template <int NS, int RB>
__device__ __forceinline__ void lsk_accum(const LskCore& p, const LskGemm& g, int et) {
  const Dims& D = p.D;
  const Pass& P = p.P;
  const int ncv = D.d >> 2, nseg = D.d >> 7;
  const ColMap m(ncv, et);
  if (m.rg >= m.nrg) return;
  const int c = m.cv * 4, lane = et & 31, rows = p.rows, d = D.d, n_out = g.n_out, max_ns = g.max_ns;
  const long long plane = g.plane;
  const float* part = p.part + c;
  float* x = P.x + c;
  const int* slot_pos = P.slot_pos;
  float* ss = p.ss + (c >> 7);
  for (int r0 = m.rg; r0 < rows; r0 += m.nrg * RB) {
    float4 w[RB][NS], xv[RB];
    int ns[RB], pos[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int row = r0 + b * m.nrg;
      pos[b] = -1;
      if (row < rows) {
        ns[b] = lsk_ns(g, row, c);
        pos[b] = __ldg(&slot_pos[row]);
        const float* pp = part + (long long)row * n_out;
#pragma unroll
        for (int k = 0; k < NS; ++k)
          if (k < max_ns) w[b][k] = ldcg4(pp + (long long)k * plane);
        xv[b] = ldcg4(x + (long long)row * d);
      }
    }
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int row = r0 + b * m.nrg;
      if (row >= rows) break;  // (uniform across the warp)
      float4 a = w[b][0];
#pragma unroll
      for (int k = 1; k < NS; ++k)
        if (k < ns[b]) add4(a, w[b][k]);
      for (int k = NS; k < ns[b]; ++k) add4(a, ldcg4(part + (long long)row * n_out + (long long)k * plane));
      add4(xv[b], a);
      const float sq = warp_sum(xv[b].x * xv[b].x + xv[b].y * xv[b].y + xv[b].z * xv[b].z + xv[b].w * xv[b].w);
      if (pos[b] >= 0) {
        *reinterpret_cast<float4*>(x + (long long)row * d) = xv[b];
        if (lane == 0) ss[(long long)row * nseg] = sq;
      }
    }
  }
}

// residual, step 2: xn = bf16(x * rsqrt(mean(x^2) + eps) * g)  (g == null: xn = x)
template <int RB>
__device__ __forceinline__ void lsk_norm(const LskCore& p, const LskGemm& g, int et) {
  const Dims& D = p.D;
  const Pass& P = p.P;
  const int ncv = D.d >> 2, nseg = D.d >> 7;
  const ColMap m(ncv, et);
  if (m.rg >= m.nrg) return;
  const int c = m.cv * 4, lane = et & 31, rows = p.rows, d = D.d;
  const bool has_ln = g.ln != nullptr;
  const float4 gg = has_ln ? ldg4(g.ln + c) : make_float4(1.f, 1.f, 1.f, 1.f);
  const float* x = P.x + c;
  const float* ssp = p.ss;
  const int* slot_pos = P.slot_pos;
  bf16* xn = reinterpret_cast<bf16*>(P.xn) + c;
  const float inv_d = 1.0f / (float)d, eps = D.eps;
  for (int r0 = m.rg; r0 < rows; r0 += m.nrg * RB) {
    float4 xv[RB];
    float sp[RB];
    int pos[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int row = r0 + b * m.nrg;
      sp[b] = 0.0f;
      pos[b] = -1;
      if (row < rows) {
        pos[b] = __ldg(&slot_pos[row]);
        xv[b] = ldcg4(x + (long long)row * d);
        if (has_ln) {  // one predicated load per lane (d <= 4096), no dependent loop
          if (lane < nseg) sp[b] = ldcg1(ssp + (long long)row * nseg + lane);
          for (int t = lane + 32; t < nseg; t += 32) sp[b] += ldcg1(ssp + (long long)row * nseg + t);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int row = r0 + b * m.nrg;
      if (row >= rows) break;
      const float s = warp_sum(sp[b]);
      if (pos[b] < 0) continue;
      float4 v = xv[b];
      if (has_ln) {
        const float inv = 1.0f / sqrtf(s * inv_d + eps);
        v.x *= inv * gg.x;
        v.y *= inv * gg.y;
        v.z *= inv * gg.z;
        v.w *= inv * gg.w;
      }
      st_bf16x4(xn + (long long)row * d, v);
    }
  }
}

// SwiGLU: act[row][f..f+3] = silu(gate) * up; gate/up interleaved per 64-feature block
template <int NS, int RB>
__device__ __forceinline__ void lsk_swiglu(const LskCore& p, const LskGemm& g, int et) {
  const Dims& D = p.D;
  const Pass& P = p.P;
  const ColMap m(D.dff >> 2, et);
  if (m.rg >= m.nrg) return;
  const int f = m.cv * 4, cg = ((f >> 6) << 7) + (f & 63), rows = p.rows, n_out = g.n_out, max_ns = g.max_ns;
  const int dff = D.dff;
  const long long plane = g.plane;
  const float* part = p.part + cg;
  const int* slot_pos = P.slot_pos;
  bf16* act = reinterpret_cast<bf16*>(P.act) + f;
  for (int r0 = m.rg; r0 < rows; r0 += m.nrg * RB) {
    float4 wg[RB][NS], wu[RB][NS];
    int ns[RB], pos[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int row = r0 + b * m.nrg;
      pos[b] = -1;
      if (row < rows) {
        ns[b] = lsk_ns(g, row, cg);
        pos[b] = __ldg(&slot_pos[row]);
        const float* pp = part + (long long)row * n_out;
#pragma unroll
        for (int k = 0; k < NS; ++k)
          if (k < max_ns) {
            wg[b][k] = ldcg4(pp + (long long)k * plane);
            wu[b][k] = ldcg4(pp + (long long)k * plane + 64);
          }
      }
    }
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      if (pos[b] < 0) continue;
      const int row = r0 + b * m.nrg;
      float4 gt = wg[b][0], up = wu[b][0];
#pragma unroll
      for (int k = 1; k < NS; ++k)
        if (k < ns[b]) {
          add4(gt, wg[b][k]);
          add4(up, wu[b][k]);
        }
      for (int k = NS; k < ns[b]; ++k) {
        add4(gt, ldcg4(part + (long long)row * n_out + (long long)k * plane));
        add4(up, ldcg4(part + (long long)row * n_out + (long long)k * plane + 64));
      }
      // silu(g) * u with MUFU exp2 / rcp (the phase runs on 4 warps per SM and is
      // issue-bound with the IEEE expf / division sequences)
      float4 a;
      a.x = gt.x * __frcp_rn(1.0f + exp2f(-1.4426950408889634f * gt.x)) * up.x;
      a.y = gt.y * __frcp_rn(1.0f + exp2f(-1.4426950408889634f * gt.y)) * up.y;
      a.z = gt.z * __frcp_rn(1.0f + exp2f(-1.4426950408889634f * gt.z)) * up.z;
      a.w = gt.w * __frcp_rn(1.0f + exp2f(-1.4426950408889634f * gt.w)) * up.w;
      st_bf16x4(act + (long long)row * dff, a);
    }
  }
}

// QKV finalize: + bias, RoPE on q/k (pairs (i, i + hd/2), per-row cos/sin
// gathered by the embed kernel), q -> P.q, k/v -> the row's KV page (window
// splice).  Column vector = (head, 4 consecutive i of the first half).
template <int NS, int RB>
__device__ __forceinline__ void lsk_qkv(const LskCore& p, const LskGemm& g, int et) {
  const Dims& D = p.D;
  const Sess& S = p.S;
  const Pass& P = p.P;
  const int half = D.hd >> 1, q4 = half >> 2;
  const ColMap m((D.nh + 2 * D.nkv) * q4, et);
  if (m.rg >= m.nrg) return;
  const int hh = m.cv / q4, i = (m.cv - hh * q4) * 4, c0 = hh * D.hd + i;
  const int rows = p.rows, n_out = g.n_out, max_ns = g.max_ns;
  const long long plane = g.plane;
  const bool rope = D.arch == 1 && hh < D.nh + D.nkv, isq = hh < D.nh;
  float4 ba = make_float4(0.f, 0.f, 0.f, 0.f), bb = ba;
  if (g.bias != nullptr) {
    ba = ldg4(g.bias + c0);
    bb = ldg4(g.bias + c0 + half);
  }
  bf16* dst0;
  if (isq) {
    dst0 = reinterpret_cast<bf16*>(P.q) + hh * D.hd + i;
  } else {
    const bool isk = hh < D.nh + D.nkv;
    const int kvh = isk ? hh - D.nh : hh - D.nh - D.nkv;
    dst0 = reinterpret_cast<bf16*>(isk ? p.st.kv_k : p.st.kv_v) +
           (long long)g.layer * S.R * S.pool * D.nkv * S.ps * D.hd + (long long)kvh * S.ps * D.hd + i;
  }
  const float* part = p.part + c0;
  const float* rr0 = P.row_rope + (long long)i * 2;
  const int* slot_pos = P.slot_pos;
  const long long* slot_kvoff = P.slot_kvoff;
  const int attn_dim = D.attn_dim;
  for (int r0 = m.rg; r0 < rows; r0 += m.nrg * RB) {
    float4 wa[RB][NS], wb[RB][NS], c01[RB], c23[RB];
    int ns[RB], pos[RB];
    long long dro[RB];
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      const int row = r0 + b * m.nrg;
      pos[b] = -1;
      if (row < rows) {
        ns[b] = lsk_ns(g, row, c0);
        pos[b] = __ldg(&slot_pos[row]);
        const float* pp = part + (long long)row * n_out;
#pragma unroll
        for (int k = 0; k < NS; ++k)
          if (k < max_ns) {
            wa[b][k] = ldcg4(pp + (long long)k * plane);
            wb[b][k] = ldcg4(pp + (long long)k * plane + half);
          }
        if (rope) {
          const float* rr = rr0 + (long long)row * half * 2;
          c01[b] = ldcg4(rr);
          c23[b] = ldcg4(rr + 4);
        }
        dro[b] = isq ? (long long)row * attn_dim : __ldg(&slot_kvoff[row]);
      }
    }
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      if (pos[b] < 0) continue;
      const int row = r0 + b * m.nrg;
      float4 a = wa[b][0], bv = wb[b][0];
#pragma unroll
      for (int k = 1; k < NS; ++k)
        if (k < ns[b]) {
          add4(a, wa[b][k]);
          add4(bv, wb[b][k]);
        }
      for (int k = NS; k < ns[b]; ++k) {
        add4(a, ldcg4(part + (long long)row * n_out + (long long)k * plane));
        add4(bv, ldcg4(part + (long long)row * n_out + (long long)k * plane + half));
      }
      add4(a, ba);
      add4(bv, bb);
      if (rope) {
        const float4 x1 = c01[b], x2 = c23[b];
        const float ax = a.x * x1.x - bv.x * x1.y, bx = bv.x * x1.x + a.x * x1.y;
        const float ay = a.y * x1.z - bv.y * x1.w, by = bv.y * x1.z + a.y * x1.w;
        const float az = a.z * x2.x - bv.z * x2.y, bz = bv.z * x2.x + a.z * x2.y;
        const float aw = a.w * x2.z - bv.w * x2.w, bw = bv.w * x2.z + a.w * x2.w;
        a = make_float4(ax, ay, az, aw);
        bv = make_float4(bx, by, bz, bw);
      }
      st_bf16x4(dst0 + dro[b], a);
      st_bf16x4(dst0 + dro[b] + half, bv);
    }
  }
}

// NS = planes unrolled in the load batch (tail loops handle more), RB rows per
// batch; one inlined variant per op (non-inlined leaves spill at the call ABI,
// and spill reloads miss the ~28 KB of L1 left next to the shared memory)
__device__ __forceinline__ void lsk_post(const LskCore& p, const LskGemm& g, int step, int et) {
  if (g.post == LSK_POST_RESIDUAL) {
    if (step == 1) lsk_norm<2>(p, g, et);
    else lsk_accum<LSK_NS_RES, LSK_RB_RES>(p, g, et);
  } else if (g.post == LSK_POST_SWIGLU) {
    lsk_swiglu<LSK_NS_SW, LSK_RB_SW>(p, g, et);
  } else {
    lsk_qkv<LSK_NS_QKV, 1>(p, g, et);
  }
}
__device__ __forceinline__ void post_bar() { asm volatile("bar.sync 2, %0;" ::"n"(LSK_POST_THREADS) : "memory"); }

// ---------------------------------------------------------------- kernel
template <int BN, int STAGES>
__global__ void __launch_bounds__(224 + LSK_POST_THREADS, 1) k_lsk(const __grid_constant__ LskParams prm) {
  using C = LskCfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ int s_skip;
  __shared__ __align__(16) LskCore sc;
  {
    const int* src = reinterpret_cast<const int*>(&prm.c);
    int* dst = reinterpret_cast<int*>(&sc);
    for (int i = threadIdx.x; i < (int)(sizeof(LskCore) / 4); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const LskCore& p = sc;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned G = gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
    }
    fence_mbar_init();
    for (int i = 0; i < p.n_gemm; ++i) {
      tma_prefetch_desc(&prm.tmA[i]);
      tma_prefetch_desc(&prm.tmB[i]);
    }
  }
  if (warp == 1) tmem_alloc(tslot, C::TCOLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  pdl_launch();

  // k-blocks this CTA streams before the dependency wait (= ring depth)
  long long total_kb = 0;
  for (int i = 0; i < p.n_gemm; ++i) total_kb += LskUnits(p.g[i], blockIdx.x).count();
  const int pre = (int)(total_kb < STAGES ? total_kb : STAGES);

  if (warp == 0) {
    // ---------------- weight producer: runs ahead through all phases
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      int stage = 0, issued = 0;
      uint32_t phase = 0;
      bool live = true;
      for (int gi = 0; gi < p.n_gemm && live; ++gi) {
        const LskGemm& g = p.g[gi];
        if ((p.flags & 1) && gi > 0 && issued > pre) {  // (diagnostic) no run-ahead across phases
          const int pp = p.g[gi - 1].post;
          grid_wait(&p.bar[3 * (gi - 1) + (pp == LSK_POST_NONE ? 0 : (pp == LSK_POST_RESIDUAL ? 2 : 1))], G);
        }
        LskUnits it(g, blockIdx.x);
        int tile, kb0, kb1, slot;
        while (live && it.next(tile, kb0, kb1, slot)) {
          const int ntile = tile % g.n_ntiles;
          for (int kb = kb0; kb < kb1; ++kb) {
            if (issued == pre) {
              pdl_wait();
              if (*p.P.skip) {
                live = false;
                break;
              }
            }
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], C::A_BYTES);
            tma_load_2d(sA + stage * C::A_BYTES, &prm.tmA[gi], &full[stage], kb * 64, ntile * 128, pol_w);
            ++issued;
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
      if (live && issued <= pre) pdl_wait();  // (tiny grids: never reached the wait above)
    }
  } else if (warp == 6) {
    // ---------------- activation producer: after each phase barrier
    if (lane == 0) {
      pdl_wait();
      const unsigned long long tb0 = globaltimer_ns();
      const int skipped = *p.P.skip;
      s_skip = skipped;
      if (skipped) {
        // complete the stages whose weight tiles are already in flight
        for (int s = 0; s < pre; ++s) mbar_arrive(&full[s]);
        for (int s = 0; s < pre; ++s) mbar_wait(&full[s], 0);
      } else {
        const uint64_t pol_x = policy_evict_last();
        int stage = 0;
        uint32_t phase = 0;
        for (int gi = 0; gi < p.n_gemm; ++gi) {
          const LskGemm& g = p.g[gi];
          if (gi > 0) {
            const int pp = p.g[gi - 1].post;
            grid_wait(&p.bar[3 * (gi - 1) + (pp == LSK_POST_NONE ? 0 : (pp == LSK_POST_RESIDUAL ? 2 : 1))], G);
          }
          fence_proxy_async_global();
          span_begin(g.tstat);
          lsk_prof(p.prof, 8 * gi + 5, tb0);
          LskUnits it(g, blockIdx.x);
          int tile, kb0, kb1, slot;
          while (it.next(tile, kb0, kb1, slot)) {
            const int chunk = tile / g.n_ntiles;
            for (int kb = kb0; kb < kb1; ++kb) {
              mbar_wait(&empty[stage], phase ^ 1);
              mbar_expect_tx(&full[stage], C::B_BYTES);
              tma_load_2d(sB + stage * C::B_BYTES, &prm.tmB[gi], &full[stage], kb * 64, chunk * BN, pol_x);
              if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      pdl_wait();
      if (!*p.P.skip) {
        constexpr uint32_t IDESC = idesc_bf16_f32(128, BN);
        int stage = 0, acc = 0;
        uint32_t phase = 0, aphase = 0;
        for (int gi = 0; gi < p.n_gemm; ++gi) {
          LskUnits it(p.g[gi], blockIdx.x);
          int tile, kb0, kb1, slot;
          while (it.next(tile, kb0, kb1, slot)) {
            mbar_wait(&tempty[acc], aphase ^ 1);
            tc_fence_after();
            const uint32_t dt = tbase + (uint32_t)(acc * BN);
            for (int kb = kb0; kb < kb1; ++kb) {
              mbar_wait(&full[stage], phase);
              tc_fence_after();
              const uint64_t ad = sdesc_sw128(smem_u32(sA + stage * C::A_BYTES));
              const uint64_t bd = sdesc_sw128(smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
              for (int k = 0; k < 4; ++k)
                tc_mma_bf16(dt, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), IDESC, (kb > kb0 || k > 0) ? 1u : 0u);
              tc_commit(&empty[stage]);
              if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
              }
            }
            tc_commit(&tfull[acc]);
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
          }
        }
      }
    }
  } else if (warp <= 5) {
    // ---------------- epilogue (warps 2-5): TMEM -> partial planes
    const int et = threadIdx.x - 64, q = warp & 3;
    pdl_wait();
    const unsigned long long t_rel = globaltimer_ns();
    unsigned long long* const prof = et == 0 ? p.prof : nullptr;
    if (prof != nullptr && blockIdx.x == 0) atomicAdd(&prof[63], 1ull);
    if (et == 0) {
      span_begin(p.tstat);
      if (blockIdx.x == 0 && p.D.klog != nullptr) {
        const unsigned long long i = atomicAdd(&p.D.klog[0], 1ull);
        if (i < (unsigned long long)p.D.klog_cap) {
          p.D.klog[1 + 2 * i] = 23ull;
          p.D.klog[2 + 2 * i] = globaltimer_ns();
        }
      }
    }
    if (!*p.P.skip) {
      int acc = 0;
      uint32_t aphase = 0;
      for (int gi = 0; gi < p.n_gemm; ++gi) {
        const LskGemm& g = p.g[gi];
        LskUnits it(g, blockIdx.x);
        int tile, kb0, kb1, slot;
        while (it.next(tile, kb0, kb1, slot)) {
          const int ntile = tile % g.n_ntiles, chunk = tile / g.n_ntiles;
          mbar_wait(&tfull[acc], aphase);
          tc_fence_after();
          const int n = ntile * 128 + q * 32 + lane;
          const int row0 = chunk * BN;
          const uint32_t taddr = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
          float* dst = p.part + (long long)slot * g.plane + n;
#pragma unroll 1
          for (int j0 = 0; j0 < BN; j0 += 32) {
            float v[32];
            tmem_ld32(taddr + j0, v);
            if (n < g.n_out) {
#pragma unroll
              for (int j = 0; j < 32; ++j) dst[(long long)(row0 + j0 + j) * g.n_out] = v[j];
            }
          }
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
          acc ^= 1;
          if (acc == 0) aphase ^= 1;
        }
        lsk_bar();
        lsk_prof(prof, 8 * gi + 0, t_rel);
        if (et == 0) {
          grid_arrive(&p.bar[3 * gi]);
          span_end(g.tstat, G);
        }
      }
    }
    if (et == 0) span_end(p.tstat, G);
  } else if (warp >= 7) {
    // ---------------- consumer ops (warps 7-14): one step (SwiGLU, QKV
    // finalize) or two with a grid barrier between them (residual: accumulate
    // + sum of squares, normalize)
    const int pt = threadIdx.x - 224;
    pdl_wait();
    const unsigned long long t_rel = globaltimer_ns();
    unsigned long long* const prof = pt == 0 ? p.prof : nullptr;
    if (!*p.P.skip) {
      for (int gi = 0; gi < p.n_gemm; ++gi) {
        const LskGemm& g = p.g[gi];
        const int steps = g.post == LSK_POST_NONE ? 0 : (g.post == LSK_POST_RESIDUAL ? 2 : 1);
        for (int step = 0; step < steps; ++step) {
          if (pt == 0) grid_wait(&p.bar[3 * gi + step], G);
          lsk_prof(prof, 8 * gi + 1 + 2 * step, t_rel);
          post_bar();
          lsk_post(p, g, step, pt);
          if (step == 0) lsk_prof(prof, 8 * gi + 6, t_rel);
          fence_proxy_async_global();
          post_bar();
          lsk_prof(prof, 8 * gi + 2 + 2 * step, t_rel);
          if (pt == 0) grid_arrive(&p.bar[3 * gi + step + 1]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, C::TCOLS);
  }
  if (threadIdx.x == 0 && !*p.P.skip) {
    // every role of this CTA is past its last wait: the last CTA out resets
    // the counters for the next launch
    __threadfence();
    if (atomicAdd(&p.bar[LSK_BAR_WORDS - 1], 1u) == G - 1) {
      for (int i = 0; i < LSK_BAR_WORDS; ++i) atomicExch(&p.bar[i], 0u);
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------- host
int lsk_stages() {
  static int st = -1;
  if (st < 0) {
    const char* e = getenv("BB_LSK_STAGES");
    st = e != nullptr ? atoi(e) : 5;
    if (st != 4 && st != 5 && st != 6 && st != 8) st = 5;
  }
  return st;
}

size_t lsk_smem(int stages) {
  switch (stages) {
    case 4: return LskCfg<64, 4>::SMEM;
    case 6: return LskCfg<64, 6>::SMEM;
    case 8: return LskCfg<64, 8>::SMEM;
    default: return LskCfg<64, 5>::SMEM;
  }
}

bool lsk_add_gemm(LskParams& p, const TcGemm& g, int post, const float* ln, const float* bias, int layer,
                  unsigned long long* tstat) {
  if (p.c.n_gemm >= LSK_MAXG || g.BN != 64 || g.p.mode != 0) return false;
  const int i = p.c.n_gemm++;
  p.tmA[i] = g.tmA;
  p.tmB[i] = g.tmB;
  LskGemm& e = p.c.g[i];
  e.n_out = g.p.n_out;
  e.K = g.p.K;
  e.n_ntiles = g.p.n_ntiles;
  e.n_chunks = g.p.n_chunks;
  e.KB = g.p.KB;
  e.G = g.grid;
  e.T = (long long)e.n_ntiles * e.n_chunks * e.KB;
  e.plane = g.p.plane;
  e.max_ns = g.max_slots;
  if (e.max_ns > 8) return false;
  e.sk = g.sk;
  e.post = post;
  e.ln = ln;
  e.bias = bias;
  e.layer = layer;
  e.tstat = tstat;
  return true;
}

template <int STAGES>
static cudaError_t lsk_launch_st(const LskParams& p, int grid, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_lsk<64, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)LskCfg<64, STAGES>::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  launch_k(k_lsk<64, STAGES>, dim3(grid), dim3(224 + LSK_POST_THREADS), (size_t)LskCfg<64, STAGES>::SMEM, s, p);
  return cudaGetLastError();
}

cudaError_t lsk_launch(const LskParams& p, int grid, cudaStream_t s) {
  switch (lsk_stages()) {
    case 4: return lsk_launch_st<4>(p, grid, s);
    case 6: return lsk_launch_st<6>(p, grid, s);
    case 8: return lsk_launch_st<8>(p, grid, s);
    default: return lsk_launch_st<5>(p, grid, s);
  }
}

}  // namespace bb
