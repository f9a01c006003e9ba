// Per-layer fused kernels of the denoiser forward (model.py:278-319 semantics,
// generalised to the LLaDA/Dream shape):
//   embed            h = emb[tok] (+ pos[p]);  xn = RMSNorm(h) (arch 1) | h
//   post_qkv         sum GEMM partial planes + bias, RoPE (arch 1), write q and
//                    the window rows' K/V into the branch's KV pages (splice)
//   post_residual    h += sum(partials);  xn = RMSNorm(h)*g | h   (next GEMM input)
//   post_gu          act = silu(gate) * up   (SwiGLU)
//   gather_head      full pass -> head slots (window rows only)
//   head_tiles_f32   fp32 mode: per-128-column (max, argmax, sumexp) from logits
//   head_reduce      combine column tiles -> conf = max prob, argmax, m, s and
//                    update the branch's probability map (h, m, s, boost)
#include "bb_common.cuh"
#include "bb_launch.cuh"
#include "bb_layers.cuh"

#ifndef POST_QKV_VEC
#define POST_QKV_VEC 1  // bf16 sessions: 4 dims per thread in k_post_qkv4
#endif
#ifndef POST_QKV_MINB
#define POST_QKV_MINB 2
#endif
#ifndef POST_QKV_NSU
#define POST_QKV_NSU 2
#endif
#ifndef POST_RES_BATCH
#define POST_RES_BATCH 1  // residual: all plane loads of a thread issued before use
#endif

namespace bb {

__device__ __forceinline__ float block_sum(float v, float* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float t = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : 0.0f;
  if (w == 0) t = warp_sum(t);
  if (threadIdx.x == 0) sh[0] = t;
  __syncthreads();
  return sh[0];
}

// ------------------------------------------------------------------ embed
template <typename T> struct Vec4;
template <> struct Vec4<float> {
  static __device__ __forceinline__ void st(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
  static __device__ __forceinline__ void st2(float* p, float*, float4 v) { *reinterpret_cast<float4*>(p) = v; }
  static __device__ __forceinline__ float4 ld(const float* p) { return *reinterpret_cast<const float4*>(p); }
};
template <> struct Vec4<__nv_bfloat16> {
  static __device__ __forceinline__ void st(__nv_bfloat16* p, float4 v) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p) = u;
  }
  // bf16x2: hi plane at p, lo plane at lo (lo = rn(v - hi)); lo == nullptr: hi only
  static __device__ __forceinline__ void st2(__nv_bfloat16* p, __nv_bfloat16* lo, float4 v) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p) = u;
    if (lo == nullptr) return;
    const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
    __nv_bfloat162 la = __floats2bfloat162_rn(v.x - fa.x, v.y - fa.y), lb = __floats2bfloat162_rn(v.z - fb.x, v.w - fb.y);
    u.x = *reinterpret_cast<uint32_t*>(&la);
    u.y = *reinterpret_cast<uint32_t*>(&lb);
    *reinterpret_cast<uint2*>(lo) = u;
  }
  static __device__ __forceinline__ float4 ld(const __nv_bfloat16* p) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
  }
};

template <typename T>
__global__ void __launch_bounds__(512) k_embed(Dims D, Pass P, const T* __restrict__ emb,
                                               const T* __restrict__ pos_emb, const float* __restrict__ ln,
                                               const float* __restrict__ rope) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 1);
  if (*P.skip) return;
  __shared__ float sh[32];
  const int row = blockIdx.x;
  int pos = P.slot_pos[row], tok = P.slot_tok[row];
  if (pos < 0) {
    pos = 0;
    tok = 0;
  }
  float* x = P.x + (long long)row * D.d;
  T* xn = reinterpret_cast<T*>(P.xn) + (long long)row * D.d;
  T* xl = P.xn_lo != nullptr ? reinterpret_cast<T*>(P.xn_lo) + (long long)row * D.d : nullptr;
  if (P.row_rope != nullptr && rope != nullptr)  // per-row RoPE table for the layer-stream QKV finalize
    for (int i = threadIdx.x; i < (D.hd >> 1); i += blockDim.x)
      *reinterpret_cast<float2*>(P.row_rope + ((long long)row * (D.hd >> 1) + i) * 2) =
          *reinterpret_cast<const float2*>(rope + ((long long)pos * (D.hd >> 1) + i) * 2);
  float ss = 0.0f;
  for (int c = threadIdx.x * 4; c < D.d; c += blockDim.x * 4) {
    float4 v = Vec4<T>::ld(emb + (long long)tok * D.d + c);
    if (D.arch == 0) {
      const float4 p = Vec4<T>::ld(pos_emb + (long long)pos * D.d + c);
      v.x += p.x;
      v.y += p.y;
      v.z += p.z;
      v.w += p.w;
    }
    *reinterpret_cast<float4*>(x + c) = v;
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  float inv = 1.0f;
  if (ln != nullptr) inv = 1.0f / sqrtf(block_sum(ss, sh) / (float)D.d + D.eps);
  for (int c = threadIdx.x * 4; c < D.d; c += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(x + c);
    if (ln != nullptr) {
      const float4 g = *reinterpret_cast<const float4*>(ln + c);
      v.x *= inv * g.x;
      v.y *= inv * g.y;
      v.z *= inv * g.z;
      v.w *= inv * g.w;
    }
    Vec4<T>::st2(xn + c, xl != nullptr ? xl + c : nullptr, v);
  }
}

// ------------------------------------------------------------------ post QKV
// CTA = (rows blockIdx.x + k * gridDim.x, group of heads of the fused q|k|v
// output); one thread per (i, i+hd/2) pair of one head.  (Batched sessions
// have thousands of rows: the grid is capped and CTAs loop over rows.)
template <typename T>
__device__ __forceinline__ void post_qkv_row(const Dims& D, const Sess& S, const Pass& P, const DevState& st,
                                             const float* __restrict__ bias, const float* __restrict__ rope, int layer,
                                             const PartRef& pr, int row) {
  const int half = D.hd >> 1;
  const int hh = blockIdx.y * (blockDim.x / half) + threadIdx.x / half, i = threadIdx.x % half;
  const bool live_hh = hh < D.nh + 2 * D.nkv;
  const int c0 = hh * D.hd + i, c1 = c0 + half;
  // session constants (piece count, bias) before the dependency wait -- except
  // in compacting sessions, whose piece counts follow this step's live rows
  if (pr.sk.rows_dyn != nullptr) {
    pdl_wait();
    if (row >= *pr.sk.rows_dyn) return;  // past the live requests' rows
  }
  const int ns = live_hh ? sk_nslots(pr.sk, row, c0) : 0;
  float ba = 0.0f, bb = 0.0f;
  if (bias != nullptr && live_hh) {
    ba = bias[c0];
    bb = bias[c1];
  }
  pdl_wait();
  klog_mark(D.klog, D.klog_cap, 2);
  // skip flag, slot, KV offset and the partial planes in one round trip
  const int skip = *P.skip, pos = P.slot_pos[row];
  const long long kvo = hh >= D.nh && live_hh ? P.slot_kvoff[row] : 0;
  float a, b;
#if POST_RES_BATCH
  if (D.hd <= 128) {
    // both halves' partial planes loaded before the adds (slot order kept);
    // c0 and c1 lie in one 128-column tile, so they share the piece count
    constexpr int NSU = 4;
    const float* pa = pr.part + (long long)row * pr.ldp + c0;
    float wa[NSU], wb[NSU];
#pragma unroll
    for (int k = 0; k < NSU; ++k)
      if (k < ns) {
        wa[k] = pa[(long long)k * pr.plane];
        wb[k] = pa[(long long)k * pr.plane + half];
      }
    if (skip || pos < 0 || !live_hh) return;
    a = wa[0];
    b = wb[0];
#pragma unroll
    for (int k = 1; k < NSU; ++k)
      if (k < ns) {
        a += wa[k];
        b += wb[k];
      }
    for (int k = NSU; k < ns; ++k) {
      a += pa[(long long)k * pr.plane];
      b += pa[(long long)k * pr.plane + half];
    }
  } else
#endif
  {
    if (skip || pos < 0 || !live_hh) return;
    a = part_sum(pr.part, pr.plane, pr.ldp, pr.sk, row, c0);
    b = part_sum(pr.part, pr.plane, pr.ldp, pr.sk, row, c1);
  }
  if (bias != nullptr) {
    a += ba;
    b += bb;
  }
  if (D.arch == 1 && hh < D.nh + D.nkv) {
    const float2 cs = *reinterpret_cast<const float2*>(rope + ((long long)pos * half + i) * 2);
    const float a2 = a * cs.x - b * cs.y, b2 = b * cs.x + a * cs.y;
    a = a2;
    b = b2;
  }
  if (hh < D.nh) {
    const long long o = (long long)row * D.attn_dim + hh * D.hd;
    T* q = reinterpret_cast<T*>(P.q) + o;
    T* ql = P.q_lo != nullptr ? reinterpret_cast<T*>(P.q_lo) + o : nullptr;
    stf2(q + i, ql != nullptr ? ql + i : nullptr, a);
    stf2(q + i + half, ql != nullptr ? ql + i + half : nullptr, b);
    return;
  }
  const bool isk = hh < D.nh + D.nkv;
  const int kvh = isk ? hh - D.nh : hh - D.nh - D.nkv;
  const long long lay = (long long)layer * S.R * S.pool * D.nkv * S.ps * D.hd;
  T* dst = reinterpret_cast<T*>(isk ? st.kv_k : st.kv_v) + lay + kvo + (long long)kvh * S.ps * D.hd;
  T* dl = st.kv_lo != 0 ? dst + st.kv_lo : nullptr;  // bf16x2: the lo pool
  stf2(dst + i, dl != nullptr ? dl + i : nullptr, a);
  stf2(dst + i + half, dl != nullptr ? dl + i + half : nullptr, b);
}

__device__ __forceinline__ void rope_rot(float& a, float& b, float c, float s) {
  const float a2 = a * c - b * s, b2 = b * c + a * s;
  a = a2;
  b = b2;
}
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void add4(float4& a, const float4& b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}

// post_qkv_row with 4 dims (and their 4 RoPE partners) per thread: float4 plane
// loads and 8-byte bf16 stores, so a thread keeps 4x the bytes in flight (large
// full passes are bound by the loads in flight).  Per element the same operations
// in the same order as post_qkv_row.
template <typename T>
__device__ __forceinline__ void post_qkv_row4(const Dims& D, const Sess& S, const Pass& P, const DevState& st,
                                              const float* __restrict__ bias, const float* __restrict__ rope, int layer,
                                              const PartRef& pr, int row) {
  const int half = D.hd >> 1, tph = half >> 2;  // threads per head
  const int hh = blockIdx.y * (blockDim.x / tph) + threadIdx.x / tph, i = (threadIdx.x % tph) * 4;
  const bool live_hh = hh < D.nh + 2 * D.nkv;
  const int c0 = hh * D.hd + i, c1 = c0 + half;
  if (pr.sk.rows_dyn != nullptr) {
    pdl_wait();
    if (row >= *pr.sk.rows_dyn) return;
  }
  const int ns = live_hh ? sk_nslots(pr.sk, row, c0) : 0;
  float4 ba = make_float4(0.0f, 0.0f, 0.0f, 0.0f), bb = ba;
  if (bias != nullptr && live_hh) {
    ba = ld4(bias + c0);
    bb = ld4(bias + c1);
  }
  pdl_wait();
  klog_mark(D.klog, D.klog_cap, 2);
  const int skip = *P.skip, pos = P.slot_pos[row];
  const long long kvo = hh >= D.nh && live_hh ? P.slot_kvoff[row] : 0;
  constexpr int NSU = POST_QKV_NSU;  // planes loaded up front
  const float* pa = pr.part + (long long)row * pr.ldp + c0;
  float4 wa[NSU], wb[NSU];
#pragma unroll
  for (int k = 0; k < NSU; ++k)
    if (k < ns) {
      wa[k] = ld4(pa + (long long)k * pr.plane);
      wb[k] = ld4(pa + (long long)k * pr.plane + half);
    }
  if (skip || pos < 0 || !live_hh) return;
  float4 a = wa[0], b = wb[0];
#pragma unroll
  for (int k = 1; k < NSU; ++k)
    if (k < ns) {
      add4(a, wa[k]);
      add4(b, wb[k]);
    }
  for (int k = NSU; k < ns; ++k) {
    add4(a, ld4(pa + (long long)k * pr.plane));
    add4(b, ld4(pa + (long long)k * pr.plane + half));
  }
  if (bias != nullptr) {
    add4(a, ba);
    add4(b, bb);
  }
  if (D.arch == 1 && hh < D.nh + D.nkv) {
    const float4 r01 = ld4(rope + ((long long)pos * half + i) * 2), r23 = ld4(rope + ((long long)pos * half + i + 2) * 2);
    rope_rot(a.x, b.x, r01.x, r01.y);
    rope_rot(a.y, b.y, r01.z, r01.w);
    rope_rot(a.z, b.z, r23.x, r23.y);
    rope_rot(a.w, b.w, r23.z, r23.w);
  }
  if (hh < D.nh) {
    const long long o = (long long)row * D.attn_dim + hh * D.hd;
    T* q = reinterpret_cast<T*>(P.q) + o;
    T* ql = P.q_lo != nullptr ? reinterpret_cast<T*>(P.q_lo) + o : nullptr;
    Vec4<T>::st2(q + i, ql != nullptr ? ql + i : nullptr, a);
    Vec4<T>::st2(q + i + half, ql != nullptr ? ql + i + half : nullptr, b);
    return;
  }
  const bool isk = hh < D.nh + D.nkv;
  const int kvh = isk ? hh - D.nh : hh - D.nh - D.nkv;
  const long long lay = (long long)layer * S.R * S.pool * D.nkv * S.ps * D.hd;
  T* dst = reinterpret_cast<T*>(isk ? st.kv_k : st.kv_v) + lay + kvo + (long long)kvh * S.ps * D.hd;
  T* dl = st.kv_lo != 0 ? dst + st.kv_lo : nullptr;  // bf16x2: the lo pool
  Vec4<T>::st2(dst + i, dl != nullptr ? dl + i : nullptr, a);
  Vec4<T>::st2(dst + i + half, dl != nullptr ? dl + i + half : nullptr, b);
}

template <typename T>
__global__ void __launch_bounds__(512) k_post_qkv(Dims D, Sess S, Pass P, DevState st, const float* __restrict__ bias,
                                                  const float* __restrict__ rope, int layer, PartRef pr) {
  pdl_launch();  // the successor launches now; our own loads follow (the first row's
                 // session constants before the dependency wait, inside post_qkv_row)
  for (int row = blockIdx.x; row < P.rows_alloc; row += gridDim.x)
    post_qkv_row<T>(D, S, P, st, bias, rope, layer, pr, row);
}

template <typename T>
__global__ void __launch_bounds__(512, POST_QKV_MINB) k_post_qkv4(Dims D, Sess S, Pass P, DevState st, const float* __restrict__ bias,
                                                   const float* __restrict__ rope, int layer, PartRef pr) {
  pdl_launch();
  for (int row = blockIdx.x; row < P.rows_alloc; row += gridDim.x)
    post_qkv_row4<T>(D, S, P, st, bias, rope, layer, pr, row);
}

// ------------------------------------------------------------------ residual (+ norm)

template <typename T>
__global__ void __launch_bounds__(512) k_post_residual(Dims D, Pass P, PartRef pr, const float* __restrict__ ln) {
  __shared__ float sh[32];
  pdl_launch();  // the successor launches now; our own loads follow
  const int row = blockIdx.x;
  float* x = P.x + (long long)row * D.d;
  T* xn = reinterpret_cast<T*>(P.xn) + (long long)row * D.d;
  T* xl = P.xn_lo != nullptr ? reinterpret_cast<T*>(P.xn_lo) + (long long)row * D.d : nullptr;
  float ss = 0.0f;
#if POST_RES_BATCH
  // d <= 4096: each thread owns <= 2 column groups.  Session constants (piece
  // counts, norm weights) are read before the dependency wait; after it the
  // skip flag, the row's slot, x and every partial plane are issued together
  // (one round trip; rows that turn out idle discard what they loaded)
  constexpr int NG = 2, NSU = 8;
  if (D.d <= NG * 4 * (int)blockDim.x) {
    float4 xv[NG], w[NG][NSU], gv[NG];
    int ns[NG], cc[NG];
    if (pr.sk.rows_dyn != nullptr) {  // compacting session: piece counts follow the live rows
      pdl_wait();
      if (row >= *pr.sk.rows_dyn) return;
    }
#pragma unroll
    for (int u = 0; u < NG; ++u) {
      cc[u] = (threadIdx.x + u * blockDim.x) * 4;
      ns[u] = cc[u] < D.d ? sk_nslots(pr.sk, row, cc[u]) : 0;
      if (ln != nullptr && cc[u] < D.d) gv[u] = *reinterpret_cast<const float4*>(ln + cc[u]);
    }
    pdl_wait();
    klog_mark(D.klog, D.klog_cap, 4);
    const int skip = *P.skip, pos = P.slot_pos[row];
#pragma unroll
    for (int u = 0; u < NG; ++u) {
      if (cc[u] < D.d) {
        const float* pp = pr.part + (long long)row * pr.ldp + cc[u];
        xv[u] = *reinterpret_cast<const float4*>(x + cc[u]);
#pragma unroll
        for (int k = 0; k < NSU; ++k)
          if (k < ns[u]) w[u][k] = *reinterpret_cast<const float4*>(pp + (long long)k * pr.plane);
      }
    }
    if (skip || pos < 0) return;
#pragma unroll
    for (int u = 0; u < NG; ++u) {
      if (cc[u] >= D.d) continue;
      float4 acc = w[u][0];
#pragma unroll
      for (int k = 1; k < NSU; ++k)
        if (k < ns[u]) {
          acc.x += w[u][k].x;
          acc.y += w[u][k].y;
          acc.z += w[u][k].z;
          acc.w += w[u][k].w;
        }
      const float* pp = pr.part + (long long)row * pr.ldp + cc[u];
      for (int k = NSU; k < ns[u]; ++k) {
        const float4 t = *reinterpret_cast<const float4*>(pp + (long long)k * pr.plane);
        acc.x += t.x;
        acc.y += t.y;
        acc.z += t.z;
        acc.w += t.w;
      }
      float4 v = xv[u];
      v.x += acc.x;
      v.y += acc.y;
      v.z += acc.z;
      v.w += acc.w;
      *reinterpret_cast<float4*>(x + cc[u]) = v;
      xv[u] = v;
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    float inv = 1.0f;
    if (ln != nullptr) inv = 1.0f / sqrtf(block_sum(ss, sh) / (float)D.d + D.eps);
#pragma unroll
    for (int u = 0; u < NG; ++u) {
      if (cc[u] >= D.d) continue;
      float4 v = xv[u];
      if (ln != nullptr) {
        const float4 g = gv[u];
        v.x *= inv * g.x;
        v.y *= inv * g.y;
        v.z *= inv * g.z;
        v.w *= inv * g.w;
      }
      Vec4<T>::st2(xn + cc[u], xl != nullptr ? xl + cc[u] : nullptr, v);
    }
    return;
  }
#endif
  pdl_wait();
  klog_mark(D.klog, D.klog_cap, 4);
  if (*P.skip) return;
  if (P.slot_pos[row] < 0) return;
  for (int c = threadIdx.x * 4; c < D.d; c += blockDim.x * 4) {
    float4 v = *reinterpret_cast<float4*>(x + c);
    const int ns = sk_nslots(pr.sk, row, c);
    const float* pp = pr.part + (long long)row * pr.ldp + c;
    float4 acc = *reinterpret_cast<const float4*>(pp);
    for (int i = 1; i < ns; ++i) {
      const float4 w = *reinterpret_cast<const float4*>(pp + (long long)i * pr.plane);
      acc.x += w.x;
      acc.y += w.y;
      acc.z += w.z;
      acc.w += w.w;
    }
    v.x += acc.x;
    v.y += acc.y;
    v.z += acc.z;
    v.w += acc.w;
    *reinterpret_cast<float4*>(x + c) = v;
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  float inv = 1.0f;
  if (ln != nullptr) inv = 1.0f / sqrtf(block_sum(ss, sh) / (float)D.d + D.eps);
  for (int c = threadIdx.x * 4; c < D.d; c += blockDim.x * 4) {
    float4 v = *reinterpret_cast<float4*>(x + c);
    if (ln != nullptr) {
      const float4 g = *reinterpret_cast<const float4*>(ln + c);
      v.x *= inv * g.x;
      v.y *= inv * g.y;
      v.z *= inv * g.z;
      v.w *= inv * g.w;
    }
    Vec4<T>::st2(xn + c, xl != nullptr ? xl + c : nullptr, v);
  }
}

// ------------------------------------------------------------------ SwiGLU
template <typename T>
__device__ __forceinline__ void post_gu_row(const Dims& D, const Pass& P, const PartRef& pr, int row) {
  const int f = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const int cg = ((f >> 6) << 7) + (f & 63);  // 4 gate features in one 64-block; up at +64
  // piece count: a session constant, read before the dependency wait (compacting
  // sessions: it follows this step's live rows)
  if (pr.sk.rows_dyn != nullptr) {
    pdl_wait();
    if (row >= *pr.sk.rows_dyn) return;
  }
  const int ns = f < D.dff ? sk_nslots(pr.sk, row, cg) : 0;
  pdl_wait();
  klog_mark(D.klog, D.klog_cap, 5);
  const float* pp = pr.part + (long long)row * pr.ldp + cg;
#if POST_RES_BATCH
  // skip flag, slot and the partial planes in one round trip (idle rows discard them)
  const int skip = *P.skip, pos = P.slot_pos[row];
  constexpr int NSU = 4;
  float4 wg[NSU], wu[NSU];
#pragma unroll
  for (int i = 0; i < NSU; ++i)
    if (i < ns) {
      wg[i] = *reinterpret_cast<const float4*>(pp + (long long)i * pr.plane);
      wu[i] = *reinterpret_cast<const float4*>(pp + (long long)i * pr.plane + 64);
    }
  if (skip || pos < 0 || f >= D.dff) return;
  float4 g = wg[0], u = wu[0];
#pragma unroll
  for (int i = 1; i < NSU; ++i)
    if (i < ns) {
      g.x += wg[i].x; g.y += wg[i].y; g.z += wg[i].z; g.w += wg[i].w;
      u.x += wu[i].x; u.y += wu[i].y; u.z += wu[i].z; u.w += wu[i].w;
    }
  for (int i = NSU; i < ns; ++i) {
#else
  if (*P.skip || P.slot_pos[row] < 0 || f >= D.dff) return;
  float4 g = *reinterpret_cast<const float4*>(pp), u = *reinterpret_cast<const float4*>(pp + 64);
  for (int i = 1; i < ns; ++i) {
#endif
    const float4 g2 = *reinterpret_cast<const float4*>(pp + (long long)i * pr.plane);
    const float4 u2 = *reinterpret_cast<const float4*>(pp + (long long)i * pr.plane + 64);
    g.x += g2.x; g.y += g2.y; g.z += g2.z; g.w += g2.w;
    u.x += u2.x; u.y += u2.y; u.z += u2.z; u.w += u2.w;
  }
  float4 a;
  a.x = g.x / (1.0f + expf(-g.x)) * u.x;
  a.y = g.y / (1.0f + expf(-g.y)) * u.y;
  a.z = g.z / (1.0f + expf(-g.z)) * u.z;
  a.w = g.w / (1.0f + expf(-g.w)) * u.w;
  const long long ao = (long long)row * D.dff + f;
  Vec4<T>::st2(reinterpret_cast<T*>(P.act) + ao, P.act_lo != nullptr ? reinterpret_cast<T*>(P.act_lo) + ao : nullptr, a);
}

// CTA = (1024 features, rows blockIdx.y + k * gridDim.y)
template <typename T>
__global__ void __launch_bounds__(256) k_post_gu(Dims D, Pass P, PartRef pr) {
  pdl_launch();  // the successor launches now; our own loads follow
  for (int row = blockIdx.y; row < P.rows_alloc; row += gridDim.y) post_gu_row<T>(D, P, pr, row);
}

// ------------------------------------------------------------------ head side
template <typename T>
__global__ void __launch_bounds__(256) k_gather_head(Dims D, Sess S, Pass full, Pass blk, Head H, int filter) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 7);
  if (*full.skip) return;
  const int slot = blockIdx.x;
  if (!H.masked[slot]) return;
  if (filter >= 0 && blk.slot_br[slot] != filter) return;
  // the full-pass row of (request, position): sequence = branch in the stacked refresh
  const int seq = full.nseq > 1 ? blk.slot_br[slot] : 0;
  const long long src = ((long long)blk.slot_req[slot] * full.nseq + seq) * S.L + blk.slot_pos[slot];
  const T* a = reinterpret_cast<const T*>(full.xn) + src * D.d;
  T* o = reinterpret_cast<T*>(blk.xn) + (long long)slot * D.d;
  for (int c = threadIdx.x; c < D.d; c += blockDim.x) o[c] = a[c];
  if (full.xn_lo != nullptr) {
    const T* al = reinterpret_cast<const T*>(full.xn_lo) + src * D.d;
    T* ol = reinterpret_cast<T*>(blk.xn_lo) + (long long)slot * D.d;
    for (int c = threadIdx.x; c < D.d; c += blockDim.x) ol[c] = al[c];
  }
}

__global__ void __launch_bounds__(128) k_head_tiles_f32(Dims D, Head H) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 8);
  if (*H.skip) return;
  const int row = blockIdx.y, vt = blockIdx.x;
  if (!H.masked[row]) return;
  __shared__ float sm[4], ss[4];
  __shared__ int sa[4];
  const int n = vt * 128 + threadIdx.x;
  float l = -INFINITY;
  if (n < D.n_out) {
    l = head_logit(H.logits[(long long)row * D.n_out + n], D.head_scale, D.spike_cut, D.spike_gain);
    if (n == H.tgt[row]) l += H.boost[row];
  }
  float m = l;
  int a = n;
  warp_argmax(m, a);
  const float e = (m == -INFINITY) ? 0.0f : expf(l - m);
  const float s = warp_sum(e);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sm[w] = m;
    sa[w] = a;
    ss[w] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm[0];
    int A = sa[0];
    for (int q = 1; q < 4; ++q)
      if (sm[q] > M) {
        M = sm[q];
        A = sa[q];
      }
    float S2 = 0.0f;
    if (M != -INFINITY)
      for (int q = 0; q < 4; ++q)
        if (sm[q] != -INFINITY) S2 += ss[q] * expf(sm[q] - M);
    H.hpart[(long long)row * D.n_vtiles + vt] = make_float4(M, __int_as_float(A), S2, 0.0f);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_head_reduce(Dims D, Sess S, Pass blk, Head H, DevState st) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 9);
  if (*H.skip) return;
  __shared__ float shm[256];
  __shared__ int sht[256];
  __shared__ float sh[32];
  const int slot = blockIdx.x;
  if (!H.masked[slot]) return;
  const float4* hp = H.hpart + (long long)slot * D.n_vtiles;
  float m = -INFINITY;
  int t0 = 0x7fffffff;
  for (int t = threadIdx.x; t < D.n_vtiles; t += blockDim.x) {
    const float mt = hp[t].x;
    if (mt > m) {
      m = mt;
      t0 = t;
    }
  }
  shm[threadIdx.x] = m;
  sht[threadIdx.x] = t0;
  __syncthreads();
  for (int o = blockDim.x >> 1; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const float m2 = shm[threadIdx.x + o];
      const int t2 = sht[threadIdx.x + o];
      if (m2 > shm[threadIdx.x] || (m2 == shm[threadIdx.x] && t2 < sht[threadIdx.x])) {
        shm[threadIdx.x] = m2;
        sht[threadIdx.x] = t2;
      }
    }
    __syncthreads();
  }
  const float M = shm[0];
  const int tb = sht[0];
  float s = 0.0f;
  for (int t = threadIdx.x; t < D.n_vtiles; t += blockDim.x) {
    const float4 v = hp[t];
    if (v.x != -INFINITY) s += v.z * expf(v.x - M);
  }
  const float Ssum = block_sum(s, sh);
  const int r = blk.slot_req[slot], b = blk.slot_br[slot], pos = blk.slot_pos[slot];
  const long long pm = ((long long)r * S.B + b) * S.L + pos;
  if (threadIdx.x == 0) {
    H.res_m[slot] = M;
    H.res_s[slot] = Ssum;
    H.res_conf[slot] = 1.0f / Ssum;
    H.res_arg[slot] = __float_as_int(hp[tb].y);
    st.pm_m[pm] = M;
    st.pm_s[pm] = Ssum;
    st.pm_boost[pm] = H.boost[slot];
    st.covered[pm] = 1;
  }
  const T* src = reinterpret_cast<const T*>(blk.xn) + (long long)slot * D.d;
  T* dst = reinterpret_cast<T*>(st.pm_h) + pm * D.d;
  for (int c = threadIdx.x; c < D.d; c += blockDim.x) dst[c] = src[c];
  if (st.pm_h_lo != nullptr) {
    const T* sl = reinterpret_cast<const T*>(blk.xn_lo) + (long long)slot * D.d;
    T* dl = reinterpret_cast<T*>(st.pm_h_lo) + pm * D.d;
    for (int c = threadIdx.x; c < D.d; c += blockDim.x) dl[c] = sl[c];
  }
}

// Materialised logits / probabilities of the last head pass (the seams'
// DenoiseOutput, model.py:160-170): per masked head slot, logit = spike(raw)
// + boost at the target column, prob = exp(logit - m) / s with the (m, s) the
// head reduction produced (so probs agree with the committed confidences).
__global__ void __launch_bounds__(128) k_head_logits(Dims D, Head H, const float* __restrict__ raw, float* logits,
                                                     float* probs) {
  pdl_enter();
  const int row = blockIdx.y;
  if (*H.skip || !H.masked[row]) return;
  const int n = blockIdx.x * 128 + threadIdx.x;
  if (n >= D.n_out) return;
  const long long i = (long long)row * D.n_out + n;
  float l = head_logit(raw[i], D.head_scale, D.spike_cut, D.spike_gain);
  if (n == H.tgt[row]) l += H.boost[row];
  logits[i] = l;
  probs[i] = expf(l - H.res_m[row]) / H.res_s[row];
}

// ------------------------------------------------------------------ launchers
#define BB_DISPATCH(D, ...)                                  \
  do {                                                       \
    if ((D).dtype == 1) {                                    \
      using T = __nv_bfloat16;                               \
      __VA_ARGS__;                                           \
    } else {                                                 \
      using T = float;                                       \
      __VA_ARGS__;                                           \
    }                                                        \
  } while (0)

cudaError_t launch_embed(const Dims& D, const Sess& S, const Pass& P, const Weights& W, cudaStream_t s) {
  BB_DISPATCH(D, (launch_k(k_embed<T>, dim3(P.rows_alloc), dim3(512), (size_t)(0), s, D, P, (const T*)W.emb, (const T*)W.pos,
                                                           D.arch == 1 ? W.ln1 : nullptr, D.arch == 1 ? W.rope : nullptr)));
  return cudaGetLastError();
}

cudaError_t launch_post_qkv(const Dims& D, const Sess& S, const Pass& P, const DevState& st, const Weights& W,
                            int layer, const PartRef& pr, cudaStream_t s) {
  const float* bias = W.bqkv != nullptr ? W.bqkv + (long long)layer * D.qkv_out : nullptr;
  const size_t smem = (size_t)D.qkv_out * sizeof(float);
  (void)smem;
  const int heads = D.nh + 2 * D.nkv, half = D.hd / 2;
  if (POST_QKV_VEC && D.dtype == 1 && half % 4 == 0 && half / 4 <= 512 && (512 % (half / 4)) == 0) {
    const int hpb = 512 / (half / 4);  // heads per CTA, 4 dims per thread
    const int gy = (heads + hpb - 1) / hpb;
    dim3 grid(P.rows_alloc < 4 * S.n_sms ? P.rows_alloc : 4 * S.n_sms, gy);
    launch_k(k_post_qkv4<__nv_bfloat16>, dim3(grid), dim3(hpb * (half / 4)), (size_t)0, s, D, S, P, st, bias, W.rope,
             layer, pr);
    return cudaGetLastError();
  }
  const int hpb = half >= 512 ? 1 : 512 / half;  // heads per CTA
  dim3 grid(P.rows_alloc < 2 * S.n_sms ? P.rows_alloc : 2 * S.n_sms, (heads + hpb - 1) / hpb);
  BB_DISPATCH(D, (launch_k(k_post_qkv<T>, dim3(grid), dim3(hpb * half), (size_t)(0), s, D, S, P, st, bias, W.rope, layer, pr)));
  return cudaGetLastError();
}

cudaError_t launch_post_residual(const Dims& D, const Pass& P, const PartRef& pr, const float* ln, cudaStream_t s) {
  BB_DISPATCH(D, (launch_k(k_post_residual<T>, dim3(P.rows_alloc), dim3(512), (size_t)(0), s, D, P, pr, ln)));
  return cudaGetLastError();
}

cudaError_t launch_post_gu(const Dims& D, const Pass& P, const PartRef& pr, cudaStream_t s) {
  dim3 grid((D.dff / 4 + 255) / 256, P.rows_alloc < 296 ? P.rows_alloc : 296);
  BB_DISPATCH(D, (launch_k(k_post_gu<T>, dim3(grid), dim3(256), (size_t)(0), s, D, P, pr)));
  return cudaGetLastError();
}

cudaError_t launch_head_logits(const Dims& D, const Pass& blk, const Head& H, float* logits, float* probs,
                               cudaStream_t s) {
  const float* raw = D.dtype == 1 ? H.raw : H.logits;
  if (raw == nullptr) return cudaErrorInvalidValue;
  launch_k(k_head_logits, dim3(D.n_vtiles, blk.rows_alloc), dim3(128), (size_t)0, s, D, H, raw, logits, probs);
  return cudaGetLastError();
}

cudaError_t launch_gather_head(const Dims& D, const Sess& S, const Pass& full, const Pass& blk, const Head& H,
                               int branch_filter, cudaStream_t s) {
  BB_DISPATCH(D, (launch_k(k_gather_head<T>, dim3(blk.rows_alloc), dim3(256), (size_t)(0), s, D, S, full, blk, H, branch_filter)));
  return cudaGetLastError();
}

cudaError_t launch_head_tiles_f32(const Dims& D, const Pass& blk, const Head& H, cudaStream_t s) {
  dim3 grid(D.n_vtiles, blk.rows_alloc);
  launch_k(k_head_tiles_f32, dim3(grid), dim3(128), (size_t)(0), s, D, H);
  return cudaGetLastError();
}

cudaError_t launch_head_reduce(const Dims& D, const Sess& S, const Pass& blk, const Head& H, const DevState& st,
                               cudaStream_t s) {
  BB_DISPATCH(D, (launch_k(k_head_reduce<T>, dim3(blk.rows_alloc), dim3(256), (size_t)(0), s, D, S, blk, H, st)));
  return cudaGetLastError();
}

}  // namespace bb
