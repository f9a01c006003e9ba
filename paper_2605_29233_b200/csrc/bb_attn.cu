// Segmented bidirectional attention over paged, shared-prefix KV.
//
// model.py:295-301: every window row (query) attends over ALL L positions of
// its branch's cache, with this step's fresh K/V already spliced into the
// window positions (post_qkv wrote them into the branch's private pages).
//
// Work item = (branch mask, run of logical pages [lp0, lp1)) built by the
// control kernel from the page tables: pages that several branches share
// (prompt after prefill, everything after a sync) form ONE item whose queries
// are the rows of all sharing branches, so a shared K/V page is streamed once
// per branch group.  CTA = (item, q-head, 32-query tile); it writes an
// unnormalised (o, m, l) partial; k_attn_combine merges the partials of the
// items covering each row (flash-decoding style LSE merge, fixed order).
#include "bb_common.cuh"
#include "bb_layers.cuh"

namespace bb {

// rows of an item: branch k in `mask` (ascending) contributes its slot range
__device__ __forceinline__ int item_row_slot(const Pass& P, const Sess& S, int r, int mask, int j) {
  for (int k = 0; k < S.B; ++k) {
    if (!((mask >> k) & 1)) continue;
    const int c = P.rng_cnt[r * MAXB + k];
    if (j < c) return P.rng_off[r * MAXB + k] + j;
    j -= c;
  }
  return -1;
}

template <typename T, int HD>
__global__ void __launch_bounds__(128) k_attn(Dims D, Sess S, Pass P, DevState st, int layer, int max_items) {
  if (*P.skip) return;
  constexpr int NPL = HD / 32;  // dims per lane
  extern __shared__ float sm[];
  float* sQ = sm;                          // [QT][HD]
  float* sK = sQ + QT * HD;                // [32][HD+1]
  float* sV = sK + 32 * (HD + 1);          // [32][HD+1]
  int* sKey = reinterpret_cast<int*>(sV + 32 * (HD + 1));  // [n_keys] element offsets (key rows)
  __shared__ int sRow[QT];

  const int r = blockIdx.x / max_items, it = blockIdx.x % max_items;
  if (it >= P.n_items[r]) return;
  const int* item = P.items + ((long long)r * max_items + it) * ITW;
  const int mask = item[0], lp0 = item[1], lp1 = item[2], rep = item[3];
  int n_rows = 0;
  for (int k = 0; k < S.B; ++k)
    if ((mask >> k) & 1) n_rows += P.rng_cnt[r * MAXB + k];
  const int row0 = blockIdx.z * QT;
  if (row0 >= n_rows) return;
  const int h = blockIdx.y, kvh = h / (D.nh / D.nkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // key table: element offset of each key row of this kv head
  const long long lay = (long long)layer * S.R * S.pool;
  long long* sKey64 = reinterpret_cast<long long*>(sKey);
  int n_keys = 0;
  for (int lp = lp0; lp < lp1; ++lp) {
    const int ks = lp_start(S, lp), ke = lp_end(S, lp);
    const long long gpage = (long long)r * S.pool + st.pt[((long long)r * S.B + rep) * S.n_lp + lp];
    const long long base = ((lay + gpage) * D.nkv + kvh) * S.ps * HD;
    for (int j = threadIdx.x; j < ke - ks; j += blockDim.x) sKey64[n_keys + j] = base + (long long)j * HD;
    n_keys += ke - ks;
  }
  if (threadIdx.x < QT) sRow[threadIdx.x] = (row0 + (int)threadIdx.x < n_rows) ? item_row_slot(P, S, r, mask, row0 + threadIdx.x) : -1;
  __syncthreads();
  const T* Qg = reinterpret_cast<const T*>(P.q);
  const float scale = D.attn_scale;
  for (int i = threadIdx.x; i < QT * HD; i += blockDim.x) {
    const int rr = i / HD, c = i % HD;
    const int slot = sRow[rr];
    sQ[i] = slot >= 0 ? ldf(Qg + (long long)slot * D.attn_dim + h * HD + c) * scale : 0.0f;
  }

  float m[8], l[8], acc[8][NPL];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    m[q] = -INFINITY;
    l[q] = 0.0f;
#pragma unroll
    for (int t = 0; t < NPL; ++t) acc[q][t] = 0.0f;
  }
  const T* Kg = reinterpret_cast<const T*>(st.kv_k);
  const T* Vg = reinterpret_cast<const T*>(st.kv_v);
  for (int k0 = 0; k0 < n_keys; k0 += 32) {
    const int nk = min(32, n_keys - k0);
    __syncthreads();
    for (int i = threadIdx.x; i < nk * HD; i += blockDim.x) {
      const int j = i / HD, c = i % HD;
      const long long o = sKey64[k0 + j] + c;
      sK[j * (HD + 1) + c] = ldf(Kg + o);
      sV[j * (HD + 1) + c] = ldf(Vg + o);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int lr = warp * 8 + q;
      if (sRow[lr] < 0) continue;  // warp-uniform
      float s = -INFINITY;
      if (lane < nk) {
        const float* qr = sQ + lr * HD;
        const float* kr = sK + lane * (HD + 1);
        float a = 0.0f;
#pragma unroll 8
        for (int c = 0; c < HD; ++c) a = fmaf(qr[c], kr[c], a);
        s = a;
      }
      const float mx = warp_max(s);
      const float mn = fmaxf(m[q], mx);
      const float corr = (m[q] == -INFINITY) ? 0.0f : expf(m[q] - mn);
      const float p = (lane < nk) ? expf(s - mn) : 0.0f;
      l[q] = l[q] * corr + warp_sum(p);
#pragma unroll
      for (int t = 0; t < NPL; ++t) acc[q][t] *= corr;
      for (int j = 0; j < nk; ++j) {
        const float pj = __shfl_sync(0xffffffffu, p, j);
        const float* vr = sV + j * (HD + 1) + lane;
#pragma unroll
        for (int t = 0; t < NPL; ++t) acc[q][t] = fmaf(pj, vr[32 * t], acc[q][t]);
      }
      m[q] = mn;
    }
  }
  // partials
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int lr = warp * 8 + q;
    if (sRow[lr] < 0) continue;
    float* o = P.apart + ((((long long)r * max_items + it) * P.item_rows + row0 + lr) * D.nh + h) * (HD + 2);
#pragma unroll
    for (int t = 0; t < NPL; ++t) o[lane + 32 * t] = acc[q][t];
    if (lane == 0) {
      o[HD] = m[q];
      o[HD + 1] = l[q];
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(128) k_attn_combine(Dims D, Sess S, Pass P, int max_items) {
  if (*P.skip) return;
  const int row = blockIdx.x;
  const int pos = P.slot_pos[row];
  if (pos < 0) return;
  const int r = P.slot_req[row], k = P.slot_br[row];
  const int j = row - P.rng_off[r * MAXB + k];
  if (j < 0 || j >= P.rng_cnt[r * MAXB + k]) return;
  const int HD = D.hd;
  const int ni = P.n_items[r];
  T* out = reinterpret_cast<T*>(P.attn) + (long long)row * D.attn_dim;
  for (int h = 0; h < D.nh; ++h) {
    // max over items covering this row
    float M = -INFINITY;
    for (int it = 0; it < ni; ++it) {
      const int mask = P.items[((long long)r * max_items + it) * ITW];
      if (!((mask >> k) & 1)) continue;
      int rii = j;
      for (int k2 = 0; k2 < k; ++k2)
        if ((mask >> k2) & 1) rii += P.rng_cnt[r * MAXB + k2];
      const float* o = P.apart + ((((long long)r * max_items + it) * P.item_rows + rii) * D.nh + h) * (HD + 2);
      M = fmaxf(M, o[HD]);
    }
    for (int c = threadIdx.x; c < HD; c += blockDim.x) {
      float acc = 0.0f, L = 0.0f;
      for (int it = 0; it < ni; ++it) {
        const int mask = P.items[((long long)r * max_items + it) * ITW];
        if (!((mask >> k) & 1)) continue;
        int rii = j;
        for (int k2 = 0; k2 < k; ++k2)
          if ((mask >> k2) & 1) rii += P.rng_cnt[r * MAXB + k2];
        const float* o = P.apart + ((((long long)r * max_items + it) * P.item_rows + rii) * D.nh + h) * (HD + 2);
        const float mi = o[HD];
        if (mi == -INFINITY) continue;
        const float w = expf(mi - M);
        acc = fmaf(o[c], w, acc);
        L = fmaf(o[HD + 1], w, L);
      }
      stf(out + h * HD + c, acc / L);
    }
  }
}

template <typename T, int HD>
static cudaError_t attn_hd(const Dims& D, const Sess& S, const Pass& P, const DevState& st, int layer,
                           int max_items, cudaStream_t s) {
  const int max_keys = P.full ? S.L : S.ch_block * S.ps;
  const size_t smem = (size_t)(QT * HD + 2 * 32 * (HD + 1)) * sizeof(float) + (size_t)max_keys * 8 + 16;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_attn<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const int max_rows = P.item_rows;
  dim3 grid(S.R * max_items, D.nh, (max_rows + QT - 1) / QT);
  k_attn<T, HD><<<grid, 128, smem, s>>>(D, S, P, st, layer, max_items);
  return cudaGetLastError();
}

cudaError_t launch_attn(const Dims& D, const Sess& S, const Pass& P, const DevState& st, int layer, cudaStream_t s) {
  const int max_items = P.full ? 1 : S.max_items;
  cudaError_t e = cudaErrorInvalidValue;
  if (D.dtype == 1) {
    using T = __nv_bfloat16;
    if (D.hd == 64) e = attn_hd<T, 64>(D, S, P, st, layer, max_items, s);
    else if (D.hd == 128) e = attn_hd<T, 128>(D, S, P, st, layer, max_items, s);
    else if (D.hd == 256) e = attn_hd<T, 256>(D, S, P, st, layer, max_items, s);
    else if (D.hd == 32) e = attn_hd<T, 32>(D, S, P, st, layer, max_items, s);
    if (e != cudaSuccess) return e;
    k_attn_combine<T><<<P.rows_alloc, 128, 0, s>>>(D, S, P, max_items);
  } else {
    using T = float;
    if (D.hd == 64) e = attn_hd<T, 64>(D, S, P, st, layer, max_items, s);
    else if (D.hd == 128) e = attn_hd<T, 128>(D, S, P, st, layer, max_items, s);
    else if (D.hd == 256) e = attn_hd<T, 256>(D, S, P, st, layer, max_items, s);
    else if (D.hd == 32) e = attn_hd<T, 32>(D, S, P, st, layer, max_items, s);
    if (e != cudaSuccess) return e;
    k_attn_combine<T><<<P.rows_alloc, 128, 0, s>>>(D, S, P, max_items);
  }
  return cudaGetLastError();
}

}  // namespace bb
