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
#include <cooperative_groups.h>
#include <stdio.h>
#include <stdlib.h>

#include <type_traits>

#include "bb_common.cuh"
#include "bb_launch.cuh"
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
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 21);
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

// ---------------------------------------------------------------------------
// bf16 tensor-core helpers (mma.sync m16n8k16, fp32 accumulate), FA2-style
// fragments: P reused from the S accumulators as the A operand of P.V, V
// fragments via ldmatrix.trans, cp.async 16-byte staging.
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void split_bf2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
  const float2 hf = __bfloat1622float2(h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(x - hf.x, y - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---------------------------------------------------------------------------
// Key lists of the tensor-core attention, built once per pass.
//
// The page tables do not change between the layers of a pass, so the walk
// over logical pages that finds, per lp, the DISTINCT physical pages among a
// key tile's branches (a page aliased by k branches -- prompt after prefill,
// everything after a sync -- is one segment with a k-bit branch mask) runs
// here once instead of in every (layer, head) attention cluster.  One CTA per
// (request, key tile); keys are emitted lp-major as (global page * ps + row,
// branch mask); akey_n = (n_keys, first key of the generation pages).
constexpr int KEY_WIN = 1 << 30;  // key-list flag: position rewritten by this step's splice

__global__ void __launch_bounds__(256) k_attn_keys(Sess S, Pass P, DevState st, int rows_per_req) {
  pdl_enter();
  extern __shared__ __align__(16) int ksm[];
  int* sPT = ksm;                         // [B][n_lp]
  int* sCnt = sPT + S.B * S.n_lp;         // [n_lp] keys per lp -> exclusive start
  int* sSeg = sCnt + S.n_lp + 1;          // [n_lp][B] physical page of segment
  int* sMsk = sSeg + S.n_lp * S.B;        // [n_lp][B] branch mask of segment
  __shared__ int s_bmask, s_tot, s_gen0;
  // full passes: row group g = (request r, sequence); the stacked refresh's
  // sequence is branch g % nseq, whose rows alone set the branch mask below
  const int g = blockIdx.x, r = P.full ? g / P.nseq : g, kz = blockIdx.y;
  const int slot_base = P.full ? g * S.L : blk_base(S, P, r);  // -1: finished request (compacting session)
  if (threadIdx.x == 0) s_bmask = 0;
  __syncthreads();
  const bool skip = *P.skip != 0;
  const int kr0 = kz << P.kz_shift, kr1 = min(rows_per_req, kr0 + (1 << P.kz_shift));
  for (int lr = kr0 + (int)threadIdx.x; lr < kr1 && !skip && slot_base >= 0; lr += blockDim.x) {
    const int sl = slot_base + lr;
    if (P.slot_pos[sl] >= 0) atomicOr(&s_bmask, 1 << P.slot_br[sl]);
  }
  for (int i = threadIdx.x; i < S.B * S.n_lp; i += blockDim.x) sPT[i] = st.pt[(long long)r * S.B * S.n_lp + i];
  __syncthreads();
  const int bmask = s_bmask;
  for (int lp = threadIdx.x; lp < S.n_lp; lp += blockDim.x) {
    int left = bmask, n = 0;
    while (left) {
      const int k = __ffs(left) - 1;
      const int phys = sPT[k * S.n_lp + lp];
      int m = 0;
      for (int k2 = k; k2 < S.B; ++k2)
        if (((left >> k2) & 1) && sPT[k2 * S.n_lp + lp] == phys) m |= 1 << k2;
      left &= ~m;
      sSeg[lp * S.B + n] = phys;
      sMsk[lp * S.B + n] = m;
      ++n;
    }
    sCnt[lp] = n * S.ps;  // segments padded to ps entries (a 64-key chunk = whole pages)
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan over lp, one warp, per-lane runs
    const int per = (S.n_lp + 31) / 32;
    const int b0 = threadIdx.x * per, b1 = min(S.n_lp, b0 + per);
    int tot = 0;
    for (int i = b0; i < b1; ++i) tot += sCnt[i];
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)threadIdx.x >= o) incl += v;
    }
    int run = incl - tot;
    for (int i = b0; i < b1; ++i) {
      const int v = sCnt[i];
      sCnt[i] = run;
      if (i == S.n_pp) s_gen0 = run;
      run += v;
    }
    if (threadIdx.x == 31) {
      s_tot = incl;
      if (S.n_pp >= S.n_lp) s_gen0 = incl;
    }
  }
  __syncthreads();
  const long long kb = (long long)g * P.n_kz + kz;
  int* out = P.akeys + kb * P.akey_cap * 2;
  // block pass: keys at a window position of one of their branches are
  // rewritten by this step's splice (KEY_WIN) -- the attention loads every
  // other key before the splice is published
  __shared__ int s_ws[MAXB], s_we[MAXB];
  if (threadIdx.x < MAXB) {
    const int k = threadIdx.x;
    const bool on = !P.full && k < S.B && ((bmask >> k) & 1);
    s_ws[k] = on ? st.br[(r * S.B + k) * B_WORDS + B_START] : 0;
    s_we[k] = on ? st.br[(r * S.B + k) * B_WORDS + B_END] : 0;
  }
  __syncthreads();
  // one thread per (lp, segment, row): lp-major emission
  for (int lp = threadIdx.x / 32; lp < S.n_lp; lp += blockDim.x / 32) {
    const int s0 = lp_start(S, lp), nk = lp_end(S, lp) - s0;
    const int base = sCnt[lp];
    const int nseg = (lp + 1 < S.n_lp ? sCnt[lp + 1] : s_tot) - base;
    for (int e = threadIdx.x & 31; e < nseg; e += 32) {
      const int j = e >> S.ps_shift, row = e & (S.ps - 1);
      const int pg = r * S.pool + sSeg[lp * S.B + j];
      const int m = row < nk ? sMsk[lp * S.B + j] : 0;  // padding rows: visible to no branch
      const int pos = s0 + row;
      bool win = false;
      for (int k = 0; k < S.B; ++k) win |= ((m >> k) & 1) && pos >= s_ws[k] && pos < s_we[k];
      out[2 * (base + e)] = pg * S.ps + row;
      out[2 * (base + e) + 1] = m | (win ? KEY_WIN : 0);
    }
  }
  if (threadIdx.x == 0) {
    P.akey_n[2 * kb] = s_tot;
    P.akey_n[2 * kb + 1] = s_gen0;
  }
}

cudaError_t launch_attn_keys(const Dims& D, const Sess& S, const Pass& P, const DevState& st, cudaStream_t s) {
  if (uses_items(D)) return cudaSuccess;
  const int rows = P.full ? S.L : S.NRq;
  const size_t smem = (size_t)(S.B * S.n_lp + S.n_lp + 1 + 2 * S.n_lp * S.B) * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_attn_keys, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  launch_k(k_attn_keys, dim3(pass_groups(S, P), P.n_kz), dim3(256), smem, s, S, P, st, rows);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Shared-prefix attention without partials (bf16 mma.sync, HD <= 128).
//
// Cluster of ATT_CS CTAs = (request, q-head, 64-row tile of the request's
// rows); each CTA of the cluster takes 1/ATT_CS of the key chunks of the
// tile's key list (k_attn_keys) and the partial softmax states are merged
// through distributed shared memory (each CTA normalises 64/ATT_CS rows).
// The rows may belong to several branches: a shared page is one run of keys
// carrying a branch mask, and row r only sees keys whose mask holds its own
// branch.  Online softmax per row, one pass, normalised output written
// directly (no split-K partials, no combine kernel).
//
// timeline runs only: per-CTA phase offsets from the PDL release, summed into
// ph[1..7] with ph[0] = CTAs (bb_session_phase_stats)
// 2^x on the SFU without exp2f's subnormal-result fix-up (results below
// 2^-126 flush to 0; the softmax weights they would be are negligible)
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void phase_mark(unsigned long long* ph, int i, unsigned long long t0) {
  if (ph != nullptr && threadIdx.x == 0) atomicAdd(&ph[i], globaltimer_ns() - t0);
}

#ifndef ATT_MERGE_H
#define ATT_MERGE_H 1  // fp16 o/l exchange in the cluster merge
#endif
#ifndef ATT_MERGE_PUSH
#define ATT_MERGE_PUSH 1  // bulk-copy push merge (needs ATT_MERGE_H)
#endif
#if ATT_MERGE_PUSH && !ATT_MERGE_H
#error ATT_MERGE_PUSH needs ATT_MERGE_H
#endif
#ifndef ATT_MMA_ILP
#define ATT_MMA_ILP 1  // independent back-to-back MMAs in the chunk loop
#endif
#ifndef ATT_KC
#define ATT_KC 64  // keys per chunk (32 measured slower: 21.6 vs 19.5 us per layer at C2)
#endif
template <int HD, int ATT_CS>
__global__ void __cluster_dims__(ATT_CS, 1, 1) __launch_bounds__(128)
    k_attn_seg(Dims D, Sess S, Pass P, DevState st, int layer, int rows_per_req) {
  klog_mark(D.klog, D.klog_cap, 24);  // (timeline) CTA 0 resident, before the dependency wait
  if (P.pf_base != nullptr && threadIdx.x == 0) {
    // this CTA's slice of the O projection's weights -> L2 (constant data: no
    // dependency; the O GEMM's TMA loads then hit L2)
    const long long n_cta = (long long)gridDim.x * gridDim.y * gridDim.z;
    const long long cta = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
    const long long per = ((P.pf_layer_bytes + n_cta - 1) / n_cta + 127) & ~127LL;
    const char* base = P.pf_base + (long long)layer * P.pf_layer_bytes;
    for (long long o = cta * per; o < min((cta + 1) * per, P.pf_layer_bytes); o += 65536) {
      const long long n = min(65536LL, min((cta + 1) * per, P.pf_layer_bytes) - o);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"((uint32_t)n) : "memory");
    }
  }
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 3);
  unsigned long long* const ats = D.klog != nullptr ? P.atstat : nullptr;  // timeline runs only
  tstat_begin(ats);
  tstat_begin(ats != nullptr ? ats + 8 : nullptr);
  tstat_end(ats != nullptr ? ats + 8 : nullptr);
  unsigned long long* const ph = ats != nullptr ? ats + 16 : nullptr;  // slot 7 (timeline runs)
  const unsigned long long t0 = ph != nullptr ? globaltimer_ns() : 0ull;
  if (ph != nullptr && threadIdx.x == 0) atomicAdd(&ph[0], 1ull);
  using bf = __nv_bfloat16;
  constexpr int KC = ATT_KC, LD = HD + 8, QR = 64;
  extern __shared__ __align__(16) uint8_t smraw[];
  bf* sQ = reinterpret_cast<bf*>(smraw);
  bf* sKb = sQ + QR * LD;       // [2][KC][LD]
  bf* sVb = sKb + 2 * KC * LD;  // [2][KC][LD]
  int2* sKeys = reinterpret_cast<int2*>(sVb + 2 * KC * LD);  // this CTA's keys
  __shared__ int sRow[QR], sBr[QR], sPos[QR];
  __shared__ int s_nk, s_gen0;
#if ATT_MERGE_PUSH
  __shared__ __align__(8) uint64_t s_mbar;  // merge: all ranks' blocks received
  if (threadIdx.x == 0) {
    mbar_init(&s_mbar, 1);
    fence_mbar_init();
    mbar_expect_tx(&s_mbar, (uint32_t)(QR * (HD + 8) * 2));
  }
#endif

  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int r = blockIdx.x / ATT_CS, h = blockIdx.y;
  const int row0 = blockIdx.z * QR;
  const int kvh = h / (D.nh / D.nkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int slot_base = P.full ? r * S.L : blk_base(S, P, r);  // (after pdl_enter) -1: finished request
  const long long kb = (long long)r * P.n_kz + (P.full ? 0 : ((blockIdx.z * 64) >> P.kz_shift));
  if (threadIdx.x < QR) {
    const int lr = row0 + threadIdx.x;
    int slot = -1, br = 0, pos = -1;
    if (lr < rows_per_req && slot_base >= 0) {
      const int sl = slot_base + lr;
      pos = P.slot_pos[sl];
      br = P.slot_br[sl];
      if (pos >= 0 && !*P.skip) slot = sl;
    }
    sRow[threadIdx.x] = slot;
    sBr[threadIdx.x] = br;
    sPos[threadIdx.x] = pos;
  } else if (threadIdx.x == QR) {
    s_nk = P.akey_n[2 * kb];
    s_gen0 = P.akey_n[2 * kb + 1];
  }
  __syncthreads();
  const int n_keys = s_nk;
  phase_mark(ph, 1, t0);
  const long long lay = (long long)layer * S.R * S.pool;
  constexpr int VPR = HD / 8;
  const bf* Kg = reinterpret_cast<const bf*>(st.kv_k);
  const bf* Vg = reinterpret_cast<const bf*>(st.kv_v);
  // keys split evenly over the cluster's CTAs (not in whole chunks: a rank with
  // one more chunk than the others would hold up the cluster merge); a partial
  // last chunk only runs the MMA tiles that hold keys
  const int k_begin = (int)((long long)n_keys * crank / ATT_CS);
  const int nk_cta = (int)((long long)n_keys * (crank + 1) / ATT_CS) - k_begin;
  const int n_chunks = (nk_cta + KC - 1) / KC;
  // this CTA's keys -> registers now, smem after the phase-A loads are out
  // (keeps the two L2 round trips overlapped)
  constexpr int KREG = 4;
  int2 kr[KREG];
  const int nkc = n_chunks * KC;
  {
    const int2* src = reinterpret_cast<const int2*>(P.akeys) + kb * P.akey_cap + k_begin;
#pragma unroll
    for (int u = 0; u < KREG; ++u) {
      const int i = threadIdx.x + u * 128;
      kr[u] = i < nk_cta ? src[i] : make_int2(0, 0);
    }
    for (int i = threadIdx.x + KREG * 128; i < nkc; i += blockDim.x) sKeys[i] = i < nk_cta ? src[i] : make_int2(0, 0);
  }
  auto store_keys = [&]() {
#pragma unroll
    for (int u = 0; u < KREG; ++u)
      if (threadIdx.x + u * 128 < nkc) sKeys[threadIdx.x + u * 128] = kr[u];
  };
  const long long kvstride = (long long)S.ps * HD;
  // ci: chunk index from this CTA's first key; part 0 = all keys, 1 = all but the
  // window keys (before the splice), 2 = only the window keys (after it)
  // element offset of key (page pg, row) for this kv head: kbase + pg * pstride
  // + row * HD (page size a power of two: shift/mask, no division per key)
  const long long kbase = (lay * D.nkv + kvh) * kvstride, pstride = (long long)D.nkv * kvstride;
  const int ps_sh = S.ps_shift, ps_mask = S.ps - 1;
  auto load_chunk = [&](int ci, int buf, int part) {
    bf* dK = sKb + buf * KC * LD;
    bf* dV = sVb + buf * KC * LD;
    const int nk = min(KC, nk_cta - ci * KC);
    for (int i = threadIdx.x; i < KC * VPR; i += blockDim.x) {
      const int j = i / VPR, v = i % VPR;
      const int2 e = sKeys[ci * KC + j];
      const bool ok = j < nk;
      const bool win = ok && (e.y & KEY_WIN) != 0;
      if ((part == 1 && win) || (part == 2 && !win)) continue;
      const long long off = kbase + (long long)(e.x >> ps_sh) * pstride + (e.x & ps_mask) * HD + v * 8;
      cp_async16(dK + j * LD + v * 8, Kg + (ok ? off : 0), ok);
      cp_async16(dV + j * LD + v * 8, Vg + (ok ? off : 0), ok);
    }
    cp_async_commit();
  };
  {
    const bf* Qg = reinterpret_cast<const bf*>(P.q);
    for (int i = threadIdx.x; i < QR * VPR; i += blockDim.x) {
      const int rr = i / VPR, v = i % VPR;
      const int slot = sRow[rr];
      cp_async16(sQ + rr * LD + v * 8, Qg + (long long)(slot >= 0 ? slot : 0) * D.attn_dim + h * HD + v * 8, slot >= 0);
    }
    cp_async_commit();
    store_keys();
    __syncthreads();  // sKeys
    if (n_chunks > 0) {
      load_chunk(0, 0, 0);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    phase_mark(ph, 5, t0);
  }
  __syncthreads();
  uint32_t qf[HD / 16][4];
  {
    const bf* q0 = sQ + (warp * 16 + g) * LD + 2 * t;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      qf[kk][0] = *reinterpret_cast<const uint32_t*>(q0 + 16 * kk);
      qf[kk][1] = *reinterpret_cast<const uint32_t*>(q0 + 8 * LD + 16 * kk);
      qf[kk][2] = *reinterpret_cast<const uint32_t*>(q0 + 16 * kk + 8);
      qf[kk][3] = *reinterpret_cast<const uint32_t*>(q0 + 8 * LD + 16 * kk + 8);
    }
  }
  const int rA = warp * 16 + g, rB = rA + 8;
  const int bA = sRow[rA] >= 0 ? sBr[rA] : 31, bB = sRow[rB] >= 0 ? sBr[rB] : 31;
  const bool warp_live = __any_sync(0xffffffffu, sRow[rA] >= 0 || sRow[rB] >= 0);
  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.0f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.0f, l1 = 0.0f;
  const float sl2 = D.attn_scale * 1.4426950408889634f;
  for (int ci = 0; ci < n_chunks; ++ci) {
    const int nk = min(KC, nk_cta - ci * KC);
    if (ci + 1 < n_chunks) {
      load_chunk(ci + 1, (ci + 1) & 1, 0);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (warp_live) {
      const int tb = ci & 1;
      const bf* sK = sKb + tb * KC * LD;
      const uint32_t sV_u = smem_u32(sVb + tb * KC * LD);
      const int2* kmask = sKeys + ci * KC;
      float s[KC / 8][4];
#pragma unroll
      for (int nt = 0; nt < KC / 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.0f;
#if ATT_MMA_ILP
      // kk outer: consecutive MMAs accumulate into different key tiles (no
      // back-to-back dependency); per tile the kk order is unchanged
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
#pragma unroll
        for (int nt = 0; nt < KC / 8; ++nt) {
          if (8 * nt >= nk) continue;  // no keys in this tile (masked to -inf below)
          const bf* k0p = sK + (8 * nt + g) * LD + 2 * t + 16 * kk;
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(k0p);
          const uint32_t b1 = *reinterpret_cast<const uint32_t*>(k0p + 8);
          mma16816(s[nt], qf[kk], b0, b1);
        }
#else
#pragma unroll
      for (int nt = 0; nt < KC / 8; ++nt) {
        if (8 * nt >= nk) continue;  // no keys in this tile (masked to -inf below)
        const bf* k0p = sK + (8 * nt + g) * LD + 2 * t;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(k0p + 16 * kk);
          const uint32_t b1 = *reinterpret_cast<const uint32_t*>(k0p + 16 * kk + 8);
          mma16816(s[nt], qf[kk], b0, b1);
        }
      }
#endif
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < KC / 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = 8 * nt + 2 * t + e;
          const int km = j < nk ? kmask[j].y : 0;
          s[nt][e] = ((km >> bA) & 1) ? s[nt][e] * sl2 : -INFINITY;
          s[nt][2 + e] = ((km >> bB) & 1) ? s[nt][2 + e] * sl2 : -INFINITY;
        }
        mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
        mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
      }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      // rows with no visible key in this chunk keep their state (mn == -inf)
      const float c0 = (m0 == -INFINITY || mn0 == -INFINITY) ? (mn0 == -INFINITY ? 1.0f : 0.0f) : ex2_ftz(m0 - mn0);
      const float c1 = (m1 == -INFINITY || mn1 == -INFINITY) ? (mn1 == -INFINITY ? 1.0f : 0.0f) : ex2_ftz(m1 - mn1);
      // rows with no visible key yet: every score is -inf, ex2(-inf - 0) = 0
      const float mb0 = mn0 == -INFINITY ? 0.0f : mn0, mb1 = mn1 == -INFINITY ? 0.0f : mn1;
      m0 = mn0;
      m1 = mn1;
      float ps0 = 0.0f, ps1 = 0.0f;
#pragma unroll
      for (int nt = 0; nt < KC / 8; ++nt) {
        s[nt][0] = ex2_ftz(s[nt][0] - mb0);
        s[nt][1] = ex2_ftz(s[nt][1] - mb0);
        s[nt][2] = ex2_ftz(s[nt][2] - mb1);
        s[nt][3] = ex2_ftz(s[nt][3] - mb1);
        ps0 += s[nt][0] + s[nt][1];
        ps1 += s[nt][2] + s[nt][3];
      }
      l0 = l0 * c0 + ps0;
      l1 = l1 * c1 + ps1;
#pragma unroll
      for (int i = 0; i < HD / 8; ++i) {
        o[i][0] *= c0;
        o[i][1] *= c0;
        o[i][2] *= c1;
        o[i][3] *= c1;
      }
#pragma unroll
      for (int kk = 0; kk < KC / 16; ++kk) {
        if (16 * kk >= nk) continue;  // P == 0 for the keys past the chunk's end
        // P = hi + lo (two bf16 parts): P.V to ~fp32 accuracy (the spike
        // epilogue amplifies attention error ~34x)
        uint32_t a[4], al[4];
        split_bf2(s[2 * kk][0], s[2 * kk][1], a[0], al[0]);
        split_bf2(s[2 * kk][2], s[2 * kk][3], a[1], al[1]);
        split_bf2(s[2 * kk + 1][0], s[2 * kk + 1][1], a[2], al[2]);
        split_bf2(s[2 * kk + 1][2], s[2 * kk + 1][3], a[3], al[3]);
        const int mi = lane >> 3, rr = lane & 7;
        const int key = 16 * kk + (mi & 1) * 8 + rr;
#if ATT_MMA_ILP
        // all hi products, then all lo products (V fragments re-read): no
        // back-to-back MMAs on one accumulator; per accumulator hi-then-lo as before
#pragma unroll
        for (int pass = 0; pass < 2; ++pass)
#pragma unroll
          for (int nt2 = 0; nt2 < HD / 8; nt2 += 2) {
            const int dim = 8 * nt2 + (mi >> 1) * 8;
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(b0, b1, b2, b3, sV_u + (uint32_t)((key * LD + dim) * 2));
            mma16816(o[nt2], pass ? al : a, b0, b1);
            mma16816(o[nt2 + 1], pass ? al : a, b2, b3);
          }
#else
#pragma unroll
        for (int nt2 = 0; nt2 < HD / 8; nt2 += 2) {
          const int dim = 8 * nt2 + (mi >> 1) * 8;
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(b0, b1, b2, b3, sV_u + (uint32_t)((key * LD + dim) * 2));
          mma16816(o[nt2], a, b0, b1);
          mma16816(o[nt2 + 1], a, b2, b3);
          mma16816(o[nt2], al, b0, b1);
          mma16816(o[nt2 + 1], al, b2, b3);
        }
#endif
      }
    }
    __syncthreads();
#if ATT_MERGE_PUSH
    // start barrier, arrive after the first chunk (wait before the push): every
    // rank's mbarrier is initialised (fence.mbarrier_init released it) and its
    // q fragments were consumed, so sQ can receive merge blocks.  Relaxed: a
    // release here would wait for the next chunk's cp.async in flight
    if (ci == 0) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
#endif
  }
#if ATT_MERGE_PUSH
  if (n_chunks == 0) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
#endif
  phase_mark(ph, 6, t0);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
#if ATT_MERGE_H
  // partial state -> own smem (reuses the K buffers): o/l as fp16 [QR][HD+8]
  // (the exchanged bytes halve; the attention output is rounded to bf16, 8x
  // coarser than these fp16 partials) and (m, l) as float2 [QR]
  constexpr int OLD = HD + 8;  // (m, l) ride in the row padding
  __half* sO = reinterpret_cast<__half*>(sKb);
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int lr = warp * 16 + g + 8 * half;
    const float lsum = half ? l1 : l0;
    const float il = lsum > 0.0f ? 1.0f / lsum : 0.0f;
#pragma unroll
    for (int nt = 0; nt < HD / 8; ++nt)
      *reinterpret_cast<__half2*>(sO + lr * OLD + 8 * nt + 2 * t) =
          __floats2half2_rn(o[nt][2 * half] * il, o[nt][2 * half + 1] * il);
    if (t == 0) *reinterpret_cast<float2*>(sO + lr * OLD + HD) = make_float2(half ? m1 : m0, lsum);
  }
#if ATT_MERGE_PUSH
  // push: rank q's rows [r*RPC, (r+1)*RPC) -> rank r's receive buffer (the dead
  // sQ: q lives in registers since the start barrier) block q, one bulk DSMEM
  // copy each, completion counted on rank r's mbarrier; no cluster barrier
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < ATT_CS) {
    constexpr uint32_t BLK = (QR / ATT_CS) * OLD * 2;
    const uint32_t dst = mapa_u32(smem_u32(sQ) + crank * BLK, threadIdx.x);
    const uint32_t bar = mapa_u32(smem_u32(&s_mbar), threadIdx.x);
    asm volatile(
        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t"
        "cp.async.bulk.commit_group;" ::"r"(dst),
        "r"(smem_u32(sO) + threadIdx.x * BLK), "r"(BLK), "r"(bar)
        : "memory");
  }
  phase_mark(ph, 2, t0);  // (timeline) start barrier / copies issued
  mbar_wait(&s_mbar, 0);
#endif
#else
  // partial state -> own smem (reuses the K buffers): o [QR][HD+4], m, l [QR]
  constexpr int OLD = HD + 4;
  float* sO = reinterpret_cast<float*>(sKb);
  float* sM = sO + QR * OLD;
  float* sL = sM + QR;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int lr = warp * 16 + g + 8 * half;
#pragma unroll
    for (int nt = 0; nt < HD / 8; ++nt)
      *reinterpret_cast<float2*>(sO + lr * OLD + 8 * nt + 2 * t) = make_float2(o[nt][2 * half], o[nt][2 * half + 1]);
    if (t == 0) {
      sM[lr] = half ? m1 : m0;
      sL[lr] = half ? l1 : l0;
    }
  }
#endif
#if !ATT_MERGE_PUSH
  cluster.sync();
  phase_mark(ph, 2, t0);  // (timeline) merge barrier passed
#endif
  // merge: this CTA normalises rows [crank*QR/CS, (crank+1)*QR/CS) across the
  // cluster; every rank's (m, l, o) is gathered into registers first
  constexpr int RPC = QR / ATT_CS;
  constexpr int V4 = HD / 4;
  constexpr int NMI = (RPC * V4 + 127) / 128;
  float mr[NMI][ATT_CS], lv[NMI][ATT_CS];
  float4 ov[NMI][ATT_CS];
#pragma unroll
  for (int k = 0; k < NMI; ++k) {
    const int i = threadIdx.x + k * 128;
    const int lr = crank * RPC + (i < RPC * V4 ? i / V4 : 0), c4 = (i % V4) * 4;
#pragma unroll
    for (int q = 0; q < ATT_CS; ++q) {
#if ATT_MERGE_H
#if ATT_MERGE_PUSH
      const __half* row = reinterpret_cast<const __half*>(sQ) + (q * RPC + lr - crank * RPC) * OLD;  // block q
#else
      const __half* row = cluster.map_shared_rank(sO + lr * OLD, q);
#endif
      const float2 ml = *reinterpret_cast<const float2*>(row + HD);
      mr[k][q] = ml.x;
      lv[k][q] = ml.y;
      const uint2 u = *reinterpret_cast<const uint2*>(row + c4);
      const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
      const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
      ov[k][q] = make_float4(a.x, a.y, b.x, b.y);  // o / l of rank q
#else
      mr[k][q] = *cluster.map_shared_rank(sM + lr, q);
      lv[k][q] = *cluster.map_shared_rank(sL + lr, q);
      ov[k][q] = *reinterpret_cast<const float4*>(cluster.map_shared_rank(sO + lr * OLD + c4, q));
#endif
    }
  }
  if (ph != nullptr) {  // (timeline) gather landed: consume one loaded value
    if (mr[0][0] == 12345.0f) __trap();
    phase_mark(ph, 3, t0);
  }
#pragma unroll
  for (int k = 0; k < NMI; ++k) {
    const int i = threadIdx.x + k * 128;
    if (i >= RPC * V4) continue;
    const int lr = crank * RPC + i / V4, c4 = (i % V4) * 4;
    const int slot = sRow[lr];
    if (slot < 0) continue;
    float M = -INFINITY;
#pragma unroll
    for (int q = 0; q < ATT_CS; ++q) M = fmaxf(M, mr[k][q]);
    float Lsum = 0.0f;
    float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
    for (int q = 0; q < ATT_CS; ++q) {
      if (mr[k][q] == -INFINITY) continue;
#if ATT_MERGE_H
      const float w = exp2f(mr[k][q] - M) * lv[k][q];  // ov holds o / l
      Lsum += w;
#else
      const float w = exp2f(mr[k][q] - M);
      Lsum += w * lv[k][q];
#endif
      acc.x += w * ov[k][q].x;
      acc.y += w * ov[k][q].y;
      acc.z += w * ov[k][q].z;
      acc.w += w * ov[k][q].w;
    }
    const float inv = 1.0f / Lsum;
    bf* out = reinterpret_cast<bf*>(P.attn) + (long long)slot * D.attn_dim + h * HD + c4;
    __nv_bfloat162 p0 = __floats2bfloat162_rn(acc.x * inv, acc.y * inv), p1 = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&p0);
    u.y = *reinterpret_cast<uint32_t*>(&p1);
    *reinterpret_cast<uint2*>(out) = u;
  }
  phase_mark(ph, 4, t0);  // (timeline) outputs stored
#if ATT_MERGE_PUSH
  // the outgoing copies must have read this CTA's staging before it exits
  if (threadIdx.x < ATT_CS) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#else
  cluster.sync();
#endif
  phase_mark(ph, 7, t0);
  tstat_end(ats);
}

template <int HD, int CS>
static cudaError_t attn_seg_launch(const Dims& D, const Sess& S, const Pass& P, const DevState& st, int layer,
                                   cudaStream_t s) {
  const int rows = P.full ? S.L : S.NRq;
  const int max_ck = (P.akey_cap + ATT_KC * CS - 1) / (ATT_KC * CS);  // chunks per CTA, upper bound
  // q + double-buffered K/V chunks (>= the merge scratch that reuses them) + keys
  const size_t kv = (size_t)4 * ATT_KC * (HD + 8) * 2, merge = (size_t)64 * (HD + 4) * 4 + 2 * 64 * 4;
  const size_t smem = (size_t)64 * (HD + 8) * 2 + (kv > merge ? kv : merge) + (size_t)max_ck * ATT_KC * 8;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_attn_seg<HD, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
  dim3 grid(pass_groups(S, P) * CS, D.nh, (rows + 63) / 64);
  launch_k(k_attn_seg<HD, CS>, dim3(grid), dim3(128), (size_t)(smem), s, D, S, P, st, layer, rows);
  return cudaGetLastError();
}

// Cluster size: the largest of 8 / 4 / 2 / 1 CTAs per (request, head, row
// tile) whose grid still fits one wave (2 CTAs of 89 KB / 238 registers per
// SM): at one request (C2 block pass, 32 heads) 8-CTA clusters split the keys;
// with several requests per session, fewer CTAs per cluster (more keys each)
// avoid running the grid in waves.  Test flags (bits 4-7) force a size.
static int att_cs(const Dims& D, const Sess& S, const Pass& P, int tflags) {
  const int forced = (tflags >> 4) & 15;
  if (forced == 8 || forced == 4 || forced == 2 || forced == 1) return forced;
  if (P.full) return 8;  // full passes: 1-CTA clusters measured 1.3% slower per C2 request
  const int rows = S.NRq;
  const long long per = (long long)pass_groups(S, P) * D.nh * ((rows + 63) / 64);
  const long long wave = 2LL * S.n_sms;
  if (per * 8 <= wave) return 8;
  if (per * 4 <= wave) return 4;
  return per * 2 <= wave ? 2 : 1;
}

// ------------------------------------------------------------------ tcgen05 block attention
// The same work split as k_attn_seg (cluster of CS CTAs per (request, head,
// 64-row key tile), keys split evenly over the ranks, (m, l, o/l) merged
// through DSMEM), with the chunk math on the 5th-gen tensor cores:
//   S[64 x 64]  = Q[64 x 128] . K_chunk^T      tcgen05.mma M=64 N=64, S in TMEM
//   O[64 x 128] += P_hi . V + P_lo . V         tcgen05.mma M=64 N=128 (V MN-major), O in TMEM
// Q, K, V and P live in shared memory in the 128-byte-swizzled UMMA layouts
// (K/V gathered per key by cp.async straight into that layout).  M=64 TMEM
// layout (measured, scripts/tc_probe.cu): rows 16w..16w+15 in lanes 0-15 of
// warp quadrant w, every column in the row's lane.  The 16x32bx2 TMEM loads
// hand lanes t and t+16 of warp w the two column halves of row 16w + t, so
// each row is split over two lanes of one warp (max / sum by one shuffle).  O is rescaled lazily (only when the row max
// grows by more than 2^8, so P stays <= 256 and its bf16 hi/lo split keeps
// ~2^-16 accuracy).
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
      "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
      "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
      "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// M=64 accumulators (16 lanes per warp quadrant): threads 0-15 get columns
// [c, c+32) of lanes 0-15, threads 16-31 columns [c+OFF, c+OFF+32)
template <int OFF>
__device__ __forceinline__ void tmem_ld16x2(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], %33;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr), "n"(OFF));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
template <int OFF>
__device__ __forceinline__ void tmem_st16x2(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x32bx2.x32.b32 [%0], %33, "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
      "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
      "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
      "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31]), "n"(OFF)
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// MN-major operand, 128B swizzle: 64-element MN atoms LBO bytes apart, 8-row
// (K) groups SBO bytes apart
__device__ __forceinline__ uint64_t sdesc_sw128_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// byte offset of 16-byte chunk c of row r in a [rows][64 bf16] SW128 tile
__device__ __forceinline__ uint32_t sw128_off(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

#ifndef ATT_TC_PLO
#define ATT_TC_PLO 1  // P.V with the bf16 lo part of P (0: hi only; measurement builds)
#endif
constexpr int ATC_QR = 64, ATC_KC = 64, ATC_HD = 128;
constexpr uint32_t ATC_SUB = 64 * 128;  // one [64 rows][64 bf16] SW128 sub-tile (bytes)

// SPLIT (bf16x2 sessions): q, K and V are hi + lo bf16 pairs (lo planes
// beside each); S = Qh.Kh + Qh.Kl + Ql.Kh and O += Ph.Vh + Pl.Vh + Ph.Vl
// (the dropped lo x lo terms are ~2^-16 relative), the cluster merge
// exchanges fp32 partials and the output is written as a hi + lo pair.
// Shared memory doubles (176 KB: one CTA per SM).
template <int CS, bool SPLIT>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(128)
    k_attn_tc(Dims D, Sess S, Pass P, DevState st, int layer, int rows_per_req) {
  klog_mark(D.klog, D.klog_cap, 24);
  if (P.pf_base != nullptr && threadIdx.x == 0) {
    // this CTA's slice of the O projection's weights -> L2 (see k_attn_seg)
    const long long n_cta = (long long)gridDim.x * gridDim.y * gridDim.z;
    const long long cta = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
    const long long per = ((P.pf_layer_bytes + n_cta - 1) / n_cta + 127) & ~127LL;
    const char* base = P.pf_base + (long long)layer * P.pf_layer_bytes;
    for (long long o = cta * per; o < min((cta + 1) * per, P.pf_layer_bytes); o += 65536) {
      const long long n = min(65536LL, min((cta + 1) * per, P.pf_layer_bytes) - o);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"((uint32_t)n) : "memory");
    }
  }
  using bf = __nv_bfloat16;
  constexpr int HD = ATC_HD, QR = ATC_QR, KC = ATC_KC;
  extern __shared__ __align__(1024) uint8_t smraw_tc[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw_tc) + 1023) & ~uintptr_t(1023));
  constexpr int NP = SPLIT ? 2 : 1;        // hi (+ lo) planes of q, K, V
  uint8_t* sQ = sm;                        // [plane][2 sub-tiles (dims 0-63, 64-127)]
  uint8_t* sK = sQ + NP * 2 * ATC_SUB;     // [plane][2 buf][2 sub]
  uint8_t* sV = sK + NP * 4 * ATC_SUB;     // [plane][2 buf][2 sub] (MN-major operand: row = key)
  uint8_t* sPh = sV + NP * 4 * ATC_SUB;    // [64 rows][64 keys] K-major
  uint8_t* sPl = sPh + ATC_SUB;
  __shared__ int sRow[QR], sBr[QR];
  __shared__ uint32_t sVis[2][32][2];  // [buf][branch][key word]: key visible to the branch
  __shared__ int2 sKr[2][ATC_KC];      // key-list ring: chunk c's keys in slot c & 1
  __shared__ int s_nk;
  __shared__ __align__(8) uint64_t mbS, mbP;
  __shared__ uint32_t s_tmem;

  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int r = blockIdx.x / CS, h = blockIdx.y;
  const int row0 = blockIdx.z * QR;
  const int kvh = h / (D.nh / D.nkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rl = 16 * warp + (lane & 15), hh = lane >> 4;  // my row, my key half (S) / dim half (O)
  int slot_base = -1;  // block pass: read after the dependency wait (compacting sessions rewrite it)
  const long long kb = (long long)r * P.n_kz + (P.full ? 0 : ((blockIdx.z * 64) >> P.kz_shift));

  if (threadIdx.x == 0) {
    mbar_init(&mbS, 1);
    mbar_init(&mbP, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&s_tmem, 256);  // S: 64 columns, O: 128 columns
  pdl_enter();
  slot_base = P.full ? r * S.L : blk_base(S, P, r);  // -1: finished request (compacting session)
  klog_mark(D.klog, D.klog_cap, 3);
  unsigned long long* const ats = D.klog != nullptr ? P.atstat : nullptr;
  tstat_begin(ats);
  unsigned long long* const ph = ats != nullptr ? ats + 16 : nullptr;  // timeline phase marks
  const unsigned long long t0 = ph != nullptr ? globaltimer_ns() : 0ull;
  if (ph != nullptr && threadIdx.x == 0) atomicAdd(&ph[0], 1ull);
  if (threadIdx.x < QR) {
    const int lr = row0 + threadIdx.x;
    int slot = -1, br = 0;
    if (lr < rows_per_req && slot_base >= 0) {
      const int sl = slot_base + lr;
      br = P.slot_br[sl];
      if (P.slot_pos[sl] >= 0 && !*P.skip) slot = sl;
    }
    sRow[threadIdx.x] = slot;
    sBr[threadIdx.x] = br;
  } else if (threadIdx.x == QR) {
    s_nk = P.akey_n[2 * kb];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tS = s_tmem, tO = s_tmem + 64;
  const int n_keys = s_nk;
  const int k_begin = (int)((long long)n_keys * crank / CS);
  const int nk_cta = (int)((long long)n_keys * (crank + 1) / CS) - k_begin;
  const int n_chunks = (nk_cta + KC - 1) / KC;
  // the key list streams through a 2-slot ring one chunk ahead of its use
  // (shared memory stays independent of the context length: 2 CTAs/SM)
  const int2* ksrc = reinterpret_cast<const int2*>(P.akeys) + kb * P.akey_cap + k_begin;
  auto key_of = [&](int c) {
    const int i = c * KC + (int)threadIdx.x;
    return i < nk_cta ? ksrc[i] : make_int2(0, 0);
  };
  int2 kreg = make_int2(0, 0);
  if (threadIdx.x < KC) {
    sKr[0][threadIdx.x] = key_of(0);
    sKr[1][threadIdx.x] = key_of(1);
    kreg = key_of(2);
  }
  const long long lay = (long long)layer * S.R * S.pool;
  const bf* Kg = reinterpret_cast<const bf*>(st.kv_k);
  const bf* Vg = reinterpret_cast<const bf*>(st.kv_v);
  const long long kvstride = (long long)S.ps * HD;
  const long long kbase = (lay * D.nkv + kvh) * kvstride, pstride = (long long)D.nkv * kvstride;
  const int ps_sh = S.ps_shift, ps_mask = S.ps - 1;
  // q rows -> SW128 sub-tiles (16-byte vector v of row rr: sub v/8, chunk v%8)
  {
    const bf* Qg = reinterpret_cast<const bf*>(P.q);
    for (int i = threadIdx.x; i < QR * 16; i += blockDim.x) {
      const int rr = i >> 4, v = i & 15;
      const int slot = sRow[rr];
      const long long qo = (long long)(slot >= 0 ? slot : 0) * D.attn_dim + h * HD + v * 8;
      cp_async16(sQ + (v >> 3) * ATC_SUB + sw128_off(rr, v & 7), Qg + qo, slot >= 0);
      if (SPLIT)
        cp_async16(sQ + 2 * ATC_SUB + (v >> 3) * ATC_SUB + sw128_off(rr, v & 7),
                   reinterpret_cast<const bf*>(P.q_lo) + qo, slot >= 0);
    }
    cp_async_commit();
  }
  __syncthreads();  // key ring
  phase_mark(ph, 1, t0);
  auto load_chunk = [&](int ci, int buf) {
    const int nk = min(KC, nk_cta - ci * KC);
    uint8_t* dK = sK + buf * 2 * ATC_SUB;
    uint8_t* dV = sV + buf * 2 * ATC_SUB;
    for (int i = threadIdx.x; i < KC * 16; i += blockDim.x) {
      const int j = i >> 4, v = i & 15;
      const int2 e = sKr[ci & 1][j];
      const bool ok = j < nk;
      const long long off = kbase + (long long)(e.x >> ps_sh) * pstride + (e.x & ps_mask) * HD + v * 8;
      const uint32_t so = (v >> 3) * ATC_SUB + sw128_off(j, v & 7);
      cp_async16(dK + so, Kg + (ok ? off : 0), ok);
      cp_async16(dV + so, Vg + (ok ? off : 0), ok);
      if (SPLIT) {  // lo pools: kv_lo elements on; lo planes 4 sub-tiles on
        cp_async16(dK + 4 * ATC_SUB + so, Kg + st.kv_lo + (ok ? off : 0), ok);
        cp_async16(dV + 4 * ATC_SUB + so, Vg + st.kv_lo + (ok ? off : 0), ok);
      }
    }
    cp_async_commit();
    // per-branch visibility bits of the chunk's keys (warp 0: keys 0-31, warp 1: 32-63)
    if (warp < 2) {
      const int j = 32 * warp + lane;
      const int m = j < nk ? sKr[ci & 1][j].y : 0;
      for (int b = 0; b < MAXB; ++b) {
        const uint32_t w = __ballot_sync(0xffffffffu, (m >> b) & 1);
        if (lane == 0) sVis[buf][b][warp] = w;
      }
      if (lane == 0) sVis[buf][31][warp] = 0u;  // rows without a slot
    }
  };
  if (n_chunks > 0) load_chunk(0, 0);
  const int br_row = sRow[rl] >= 0 ? sBr[rl] : 31;  // bit 31 is never set: no visible key
  const float sl2 = D.attn_scale * 1.4426950408889634f;
  float m_ref = -INFINITY, l_part = 0.0f;
  constexpr uint32_t IDS = idesc_bf16_f32(64, 64);
  constexpr uint32_t IDO = idesc_bf16_f32(64, 128) | (1u << 16);  // B (V) MN-major
  const uint32_t tl = (uint32_t)(32 * warp) << 16;                 // my TMEM lane quadrant
  for (int ci = 0; ci < n_chunks; ++ci) {
    const int buf = ci & 1;
    const int nk = min(KC, nk_cta - ci * KC);
    // loaders: this chunk (and q) landed -> visible to the tensor core, then
    // the next chunk's gather (its buffer was last read by S and P.V of ci-1)
    cp_async_wait<0>();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    // P.V of chunk ci-1 done (every phase is observed in order: parity waits
    // must never fall two phases behind): its K/V buffer is free
    if (ci > 0) mbar_wait(&mbP, (ci - 1) & 1);
    if (ci + 1 < n_chunks) load_chunk(ci + 1, buf ^ 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK + buf * 2 * ATC_SUB);
#pragma unroll
      for (int ks = 0; ks < HD / 16; ++ks) {
        const uint32_t sub = (ks >> 2) * ATC_SUB, ko = (ks & 3) * 32;
        tc_mma_bf16(tS, sdesc_sw128(q0 + sub + ko), sdesc_sw128(k0 + sub + ko), IDS, ks > 0 ? 1u : 0u);
      }
      if (SPLIT) {  // + Qh.Kl + Ql.Kh
        const uint32_t ql = q0 + 2 * ATC_SUB, kl = k0 + 4 * ATC_SUB;
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) {
          const uint32_t sub = (ks >> 2) * ATC_SUB, ko = (ks & 3) * 32;
          tc_mma_bf16(tS, sdesc_sw128(q0 + sub + ko), sdesc_sw128(kl + sub + ko), IDS, 1u);
          tc_mma_bf16(tS, sdesc_sw128(ql + sub + ko), sdesc_sw128(k0 + sub + ko), IDS, 1u);
        }
      }
      tc_commit(&mbS);
    }
    if (ci == 0) phase_mark(ph, 5, t0);  // (timeline) chunk 0 landed
    mbar_wait(&mbS, ci & 1);  // S(ci) done, and with it P.V of chunk ci-1
    tc_fence_after();
    if (ci == 0) phase_mark(ph, 2, t0);  // (timeline) first S done
    float s[32];
    tmem_ld16x2<32>(tS + tl, s);  // row rl, keys 32*hh + [0, 32)
    const uint32_t vw = sVis[buf][br_row][hh];
    float mx4[4] = {m_ref, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      s[c] = ((vw >> c) & 1u) ? s[c] * sl2 : -INFINITY;
      mx4[c & 3] = fmaxf(mx4[c & 3], s[c]);
    }
    float m_new = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
    m_new = fmaxf(m_new, __shfl_xor_sync(0xffffffffu, m_new, 16));
    const bool grow = m_new > m_ref + 8.0f;  // (also the first visible key: m_ref = -inf)
    const float f = !grow ? 1.0f : (m_ref == -INFINITY ? 0.0f : ex2_ftz(m_ref - m_new));
    // O rows that held visible keys are rescaled in TMEM; tcgen05.ld/st are
    // warp-collective, so the whole warp takes the branch (f = 1 elsewhere)
    if (ci > 0 && __any_sync(0xffffffffu, grow && m_ref != -INFINITY)) {
      float o[32];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        tmem_ld16x2<64>(tO + tl + 32 * q, o);
#pragma unroll
        for (int c = 0; c < 32; ++c) o[c] *= f;
        tmem_st16x2<64>(tO + tl + 32 * q, o);
      }
    }
    if (grow) {
      l_part *= f;
      m_ref = m_new;
    }
    const float mb = m_ref == -INFINITY ? 0.0f : m_ref;
    // P = 2^(s - m_ref) as bf16 hi + lo, my 32 keys of row rl: 4 x 16-byte chunks
    {
      float ls[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int c8 = 0; c8 < 4; ++c8) {
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p0 = ex2_ftz(s[8 * c8 + 2 * e] - mb), p1 = ex2_ftz(s[8 * c8 + 2 * e + 1] - mb);
          ls[e] += p0 + p1;
          split_bf2(p0, p1, hi[e], lo[e]);
        }
        const uint32_t off = sw128_off(rl, 4 * hh + c8);
        *reinterpret_cast<uint4*>(sPh + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        if (ATT_TC_PLO || SPLIT) *reinterpret_cast<uint4*>(sPl + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
      l_part += (ls[0] + ls[1]) + (ls[2] + ls[3]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    // keys of chunk ci+2 into the slot chunk ci's keys held (read by
    // load_chunk(ci), done); visible after this barrier, used at ci+1's top
    if (threadIdx.x < KC) {
      sKr[ci & 1][threadIdx.x] = kreg;
      kreg = key_of(ci + 3);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t v0 = smem_u32(sV + buf * 2 * ATC_SUB), pa = smem_u32(sPh), pl = smem_u32(sPl);
#pragma unroll
      for (int kk = 0; kk < KC / 16; ++kk) {
        const uint64_t bd = sdesc_sw128_mn(v0 + kk * 2048, ATC_SUB, 1024);
        tc_mma_bf16(tO, sdesc_sw128(pa + kk * 32), bd, IDO, (ci > 0 || kk > 0) ? 1u : 0u);
        if (ATT_TC_PLO || SPLIT) tc_mma_bf16(tO, sdesc_sw128(pl + kk * 32), bd, IDO, 1u);
        if (SPLIT)  // + Ph.Vl
          tc_mma_bf16(tO, sdesc_sw128(pa + kk * 32), sdesc_sw128_mn(v0 + 4 * ATC_SUB + kk * 2048, ATC_SUB, 1024), IDO,
                      1u);
      }
      tc_commit(&mbP);
    }
  }
  // partial state (m_ref, l, o / l) of my row half -> fp16 (SPLIT: fp32)
  // staging in the (now idle) K buffers: [QR][HD + 8] elements, (m, l) in the
  // row padding
  constexpr int OLD = HD + 8;
  using ST = typename std::conditional<SPLIT, float, __half>::type;
  ST* sO = reinterpret_cast<ST*>(sK);
  phase_mark(ph, 6, t0);
  if (n_chunks > 0) mbar_wait(&mbP, (n_chunks - 1) & 1);
  tc_fence_after();
  __syncthreads();
  phase_mark(ph, 3, t0);  // (timeline) last P.V done

  {
    const float lsum = l_part + __shfl_xor_sync(0xffffffffu, l_part, 16);
    const float il = lsum > 0.0f ? 1.0f / lsum : 0.0f;
    float o[32];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (n_chunks > 0) {
        tmem_ld16x2<64>(tO + tl + 32 * q, o);  // dims 64*hh + 32*q + [0, 32)
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) o[c] = 0.0f;
      }
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        if constexpr (SPLIT)
          *reinterpret_cast<float2*>(sO + rl * OLD + 64 * hh + 32 * q + c) = make_float2(o[c] * il, o[c + 1] * il);
        else
          *reinterpret_cast<__half2*>(sO + rl * OLD + 64 * hh + 32 * q + c) = __floats2half2_rn(o[c] * il, o[c + 1] * il);
      }
    }
    if (hh == 0) *reinterpret_cast<float2*>(sO + rl * OLD + HD) = make_float2(m_ref, lsum);
  }
  tc_fence_before();
  cluster.sync();
  // merge rows [crank*RPC, (crank+1)*RPC) over the cluster (pull; fixed rank order)
  constexpr int RPC = QR / CS, V4 = HD / 4, NMI = (RPC * V4 + 127) / 128;
#pragma unroll
  for (int k = 0; k < NMI; ++k) {
    const int i = threadIdx.x + k * 128;
    if (i >= RPC * V4) continue;
    const int lr = crank * RPC + i / V4, c4 = (i % V4) * 4;
    const int slot = sRow[lr];
    float mr[CS], lv[CS];
    float4 ov[CS];
#pragma unroll
    for (int q = 0; q < CS; ++q) {
      const ST* row = cluster.map_shared_rank(sO + lr * OLD, q);
      const float2 ml = *reinterpret_cast<const float2*>(row + HD);
      mr[q] = ml.x;
      lv[q] = ml.y;
      if constexpr (SPLIT) {
        ov[q] = *reinterpret_cast<const float4*>(row + c4);
      } else {
        const uint2 u = *reinterpret_cast<const uint2*>(row + c4);
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
        const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
        ov[q] = make_float4(a.x, a.y, b.x, b.y);
      }
    }
    if (slot < 0) continue;
    float M = -INFINITY;
#pragma unroll
    for (int q = 0; q < CS; ++q) M = fmaxf(M, mr[q]);
    float Lsum = 0.0f;
    float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
    for (int q = 0; q < CS; ++q) {
      if (mr[q] == -INFINITY || lv[q] <= 0.0f) continue;
      const float w = ex2_ftz(mr[q] - M) * lv[q];
      Lsum += w;
      acc.x += w * ov[q].x;
      acc.y += w * ov[q].y;
      acc.z += w * ov[q].z;
      acc.w += w * ov[q].w;
    }
    const float inv = Lsum > 0.0f ? 1.0f / Lsum : 0.0f;
    const long long oo = (long long)slot * D.attn_dim + h * HD + c4;
    bf* out = reinterpret_cast<bf*>(P.attn) + oo;
    const float4 y = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    __nv_bfloat162 p0 = __floats2bfloat162_rn(y.x, y.y), p1 = __floats2bfloat162_rn(y.z, y.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&p0);
    u.y = *reinterpret_cast<uint32_t*>(&p1);
    *reinterpret_cast<uint2*>(out) = u;
    if (SPLIT) {  // lo = rn(y - hi)
      const float2 f0 = __bfloat1622float2(p0), f1 = __bfloat1622float2(p1);
      __nv_bfloat162 l0 = __floats2bfloat162_rn(y.x - f0.x, y.y - f0.y), l1 = __floats2bfloat162_rn(y.z - f1.x, y.w - f1.y);
      u.x = *reinterpret_cast<uint32_t*>(&l0);
      u.y = *reinterpret_cast<uint32_t*>(&l1);
      *reinterpret_cast<uint2*>(reinterpret_cast<bf*>(P.attn_lo) + oo) = u;
    }
  }
  phase_mark(ph, 4, t0);  // (timeline) merged outputs stored
  cluster.sync();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(s_tmem, 256);
  }
  phase_mark(ph, 7, t0);
  tstat_end(ats);
}

template <int CS, bool SPLIT>
static cudaError_t attn_tc_launch(const Dims& D, const Sess& S, const Pass& P, const DevState& st, int layer,
                                  cudaStream_t s) {
  const int rows = P.full ? S.L : S.NRq;
  // keys stream through a static ring: q 2, K 4, V 4 sub-tiles per plane + P hi/lo
  const size_t smem = 1024 + (size_t)((SPLIT ? 2 : 1) * 10 + 2) * ATC_SUB;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_attn_tc<CS, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
  dim3 grid(pass_groups(S, P) * CS, D.nh, (rows + ATC_QR - 1) / ATC_QR);
  launch_k(k_attn_tc<CS, SPLIT>, dim3(grid), dim3(128), (size_t)(smem), s, D, S, P, st, layer, rows);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ warp-specialized tcgen05 attention
// k_attn_fa: the k_attn_tc work split and math (M = 64 query rows, 64-key
// chunks, S / O in TMEM, P as bf16 hi + lo, DSMEM cluster merge) with the
// chunk pipeline taken apart into roles that run concurrently:
//   warp 4 (producer): per chunk, the keys' branch-visibility words and the
//     chunk's four 16-key KV pages -> an NS-deep shared-memory ring by TMA
//     (128-byte-swizzled boxes of one page x 64 dims, complete_tx mbarrier);
//     the key list pads every page segment to 16 entries (k_attn_keys), so a
//     chunk is exactly four whole pages.
//   warp 5 lane 0 (MMA issuer): S(ci) = Q.K(ci)^T into one of two TMEM S
//     buffers as soon as the chunk landed and that buffer was read, THEN
//     O += P(ci-1).V(ci-1) -- the score MMA of the next chunk overlaps the
//     softmax of the current one; the P.V commit frees the ring slot.
//     (Issuing P.V by readiness instead measured 8% slower here at C2; it is
//     what k_attn_fa128's single-P-buffer instance does.)
//   warps 0-3 (softmax): row max / lazy O rescale / P = 2^(s - m) as bf16
//     hi + lo, exactly as k_attn_tc.
// No __syncthreads in the chunk loop; every hand-off is an mbarrier.
// SPLIT (bf16x2 sessions): q / K / V hi + lo planes (the lo pools through
// their own TMA views), S = Qh.Kh + Qh.Kl + Ql.Kh, O += Ph.Vh + Pl.Vh + Ph.Vl,
// fp32 cluster merge, hi + lo output (see k_attn_tc).
constexpr int AFA_THREADS = 192;

template <int CS, int NS, bool SPLIT>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(AFA_THREADS)
    k_attn_fa(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
              const __grid_constant__ CUtensorMap tmKl, const __grid_constant__ CUtensorMap tmVl, Dims D, Sess S,
              Pass P, DevState st, int layer, int rows_per_req) {
  klog_mark(D.klog, D.klog_cap, 24);
  if (P.pf_base != nullptr && threadIdx.x == 0) {
    // this CTA's slice of the O projection's weights -> L2 (HBM is not saturated by the attention)
    const long long n_cta = (long long)gridDim.x * gridDim.y * gridDim.z;
    const long long cta = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
    const long long per = ((P.pf_layer_bytes + n_cta - 1) / n_cta + 127) & ~127LL;
    const char* base = P.pf_base + (long long)layer * P.pf_layer_bytes;
    for (long long o = cta * per; o < min((cta + 1) * per, P.pf_layer_bytes); o += 65536) {
      const long long n = min(65536LL, min((cta + 1) * per, P.pf_layer_bytes) - o);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"((uint32_t)n) : "memory");
    }
  }
  using bf = __nv_bfloat16;
  constexpr int HD = ATC_HD, QR = ATC_QR, KC = ATC_KC;
  constexpr int NP = SPLIT ? 2 : 1;             // hi (+ lo) planes
  constexpr uint32_t STAGE = NP * 4 * ATC_SUB;  // [K hi 2 sub, V hi 2 sub (, K lo 2, V lo 2)]
  extern __shared__ __align__(1024) uint8_t smraw_fa[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw_fa) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;                       // [plane][2 sub-tiles (dims 0-63, 64-127)]
  uint8_t* sKV = sQ + NP * 2 * ATC_SUB;   // [NS] stages
  uint8_t* sPh = sKV + NS * STAGE;   // [64 rows][64 keys] K-major
  uint8_t* sPl = sPh + ATC_SUB;
  __shared__ int sRow[QR], sBr[QR];
  __shared__ uint32_t sVis[NS][32][2];  // [slot][branch][key word]
  __shared__ int s_nk;
  __shared__ __align__(8) uint64_t kfull[NS], kempty[NS], sfull[2], sfree[2], pfull, pvdone, qready;
  __shared__ uint32_t s_tmem;

  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int r = blockIdx.x / CS, h = blockIdx.y;
  const int row0 = blockIdx.z * QR;
  const int kvh = h / (D.nh / D.nkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int slot_base = -1;  // block pass: read after the dependency wait (compacting sessions rewrite it)
  const long long kb = (long long)r * P.n_kz + (P.full ? 0 : ((blockIdx.z * 64) >> P.kz_shift));

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kfull[i], 1);
      mbar_init(&kempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sfree[i], 4);
    }
    mbar_init(&pfull, 4);
    mbar_init(&pvdone, 1);
    mbar_init(&qready, 128);
    fence_mbar_init();
  }
  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    if (SPLIT) {
      tma_prefetch_desc(&tmKl);
      tma_prefetch_desc(&tmVl);
    }
  }
  if (warp == 5) tmem_alloc(&s_tmem, 256);  // S0, S1: 64 columns each; O: 128 columns
  pdl_enter();
  slot_base = P.full ? r * S.L : blk_base(S, P, r);  // -1: finished request (compacting session)
  klog_mark(D.klog, D.klog_cap, 3);
  unsigned long long* const ats = D.klog != nullptr ? P.atstat : nullptr;
  tstat_begin(ats);
  if (threadIdx.x < QR) {
    const int lr = row0 + threadIdx.x;
    int slot = -1, br = 0;
    if (lr < rows_per_req && slot_base >= 0) {
      const int sl = slot_base + lr;
      br = P.slot_br[sl];
      if (P.slot_pos[sl] >= 0 && !*P.skip) slot = sl;
    }
    sRow[threadIdx.x] = slot;
    sBr[threadIdx.x] = br;
  } else if (threadIdx.x == QR) {
    s_nk = P.akey_n[2 * kb];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tS0 = s_tmem, tO = s_tmem + 128;
  // keys split over the cluster in whole chunks (a chunk = four whole pages)
  const int n_keys = s_nk;
  const int nc_all = (n_keys + KC - 1) / KC;
  const int c_begin = (int)((long long)nc_all * crank / CS);
  const int n_chunks = (int)((long long)nc_all * (crank + 1) / CS) - c_begin;
  const int k_begin = c_begin * KC;
  const int2* ksrc = reinterpret_cast<const int2*>(P.akeys) + kb * P.akey_cap + k_begin;
  const int nk_cta = min(n_keys - k_begin, n_chunks * KC);

  if (warp == 4) {
    // ---------------- producer: visibility words + TMA page loads.  The key
    // entries of chunk ci+1 are read (global) while chunk ci waits for its
    // ring slot, so the key-list latency stays off the load chain.
    const uint64_t pol = policy_evict_normal();  // the prompt's pages are re-read by other row tiles
    const int lay_rows = layer * S.R * S.pool;   // (layer, page) -> row of the [rows][hd] KV view
    auto entries = [&](int ci, int2& e0, int2& e1) {
      const int i0 = ci * KC + lane, i1 = i0 + 32;
      e0 = (ci < n_chunks && i0 < nk_cta) ? ksrc[i0] : make_int2(0, 0);
      e1 = (ci < n_chunks && i1 < nk_cta) ? ksrc[i1] : make_int2(0, 0);
    };
    int2 e0, e1, n0, n1;
    entries(0, e0, e1);
    for (int ci = 0; ci < n_chunks; ++ci) {
      const int slot = ci % NS;
      uint32_t vis[2 * MAXB];
#pragma unroll
      for (int b = 0; b < MAXB; ++b) {
        vis[2 * b] = __ballot_sync(0xffffffffu, b < S.B && ((e0.y >> b) & 1));
        vis[2 * b + 1] = __ballot_sync(0xffffffffu, b < S.B && ((e1.y >> b) & 1));
      }
      // global page of each 16-key group (entries 0, 16, 32, 48 of the chunk)
      const int pg0 = __shfl_sync(0xffffffffu, e0.x, 0) >> 4, pg1 = __shfl_sync(0xffffffffu, e0.x, 16) >> 4;
      const int pg2 = __shfl_sync(0xffffffffu, e1.x, 0) >> 4, pg3 = __shfl_sync(0xffffffffu, e1.x, 16) >> 4;
      entries(ci + 1, n0, n1);
      if (ci >= NS) mbar_wait(&kempty[slot], ((ci / NS) - 1) & 1);
      if (lane == 0) {
#pragma unroll
        for (int b = 0; b < MAXB; ++b) {
          sVis[slot][b][0] = vis[2 * b];
          sVis[slot][b][1] = vis[2 * b + 1];
        }
        sVis[slot][31][0] = 0u;  // rows without a slot
        sVis[slot][31][1] = 0u;
        const int nk = min(KC, nk_cta - ci * KC);
        // groups past the chunk's keys re-load group 0's page (finite data, masked out)
        const int pgs[4] = {pg0, nk > 16 ? pg1 : pg0, nk > 32 ? pg2 : pg0, nk > 48 ? pg3 : pg0};
        uint8_t* dst = sKV + slot * STAGE;
        mbar_expect_tx(&kfull[slot], STAGE);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int row = ((lay_rows + pgs[g]) * D.nkv + kvh) * 16;
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {
            tma_load_2d(dst + sub * ATC_SUB + g * 2048, &tmK, &kfull[slot], sub * 64, row, pol);
            tma_load_2d(dst + (2 + sub) * ATC_SUB + g * 2048, &tmV, &kfull[slot], sub * 64, row, pol);
            if (SPLIT) {
              tma_load_2d(dst + (4 + sub) * ATC_SUB + g * 2048, &tmKl, &kfull[slot], sub * 64, row, pol);
              tma_load_2d(dst + (6 + sub) * ATC_SUB + g * 2048, &tmVl, &kfull[slot], sub * 64, row, pol);
            }
          }
        }
      }
      e0 = n0;
      e1 = n1;
      __syncwarp();
    }
  } else if (warp == 5) {
    // ---------------- MMA issuer
    if (lane == 0 && n_chunks > 0) {
      constexpr uint32_t IDS = idesc_bf16_f32(64, 64);
      constexpr uint32_t IDO = idesc_bf16_f32(64, 128) | (1u << 16);  // B (V) MN-major
      mbar_wait(&qready, 0);
      tc_fence_after();
      const uint32_t q0 = smem_u32(sQ), pa = smem_u32(sPh), pl = smem_u32(sPl);
      for (int ci = 0; ci <= n_chunks; ++ci) {
        if (ci < n_chunks) {
          const int slot = ci % NS, sb = ci & 1;
          mbar_wait(&kfull[slot], (ci / NS) & 1);
          if (ci >= 2) mbar_wait(&sfree[sb], ((ci >> 1) - 1) & 1);
          tc_fence_after();
          const uint32_t k0 = smem_u32(sKV + slot * STAGE);
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks) {
            const uint32_t sub = (ks >> 2) * ATC_SUB, ko = (ks & 3) * 32;
            tc_mma_bf16(tS0 + 64 * sb, sdesc_sw128(q0 + sub + ko), sdesc_sw128(k0 + sub + ko), IDS,
                        ks > 0 ? 1u : 0u);
          }
          if (SPLIT) {  // + Qh.Kl + Ql.Kh
            const uint32_t ql = q0 + 2 * ATC_SUB, kl = k0 + 4 * ATC_SUB;
#pragma unroll
            for (int ks = 0; ks < HD / 16; ++ks) {
              const uint32_t sub = (ks >> 2) * ATC_SUB, ko = (ks & 3) * 32;
              tc_mma_bf16(tS0 + 64 * sb, sdesc_sw128(q0 + sub + ko), sdesc_sw128(kl + sub + ko), IDS, 1u);
              tc_mma_bf16(tS0 + 64 * sb, sdesc_sw128(ql + sub + ko), sdesc_sw128(k0 + sub + ko), IDS, 1u);
            }
          }
          tc_commit(&sfull[sb]);
        }
        if (ci >= 1) {
          const int pc = ci - 1, pslot = pc % NS;
          mbar_wait(&pfull, pc & 1);
          tc_fence_after();
          const uint32_t v0 = smem_u32(sKV + pslot * STAGE + 2 * ATC_SUB);
#pragma unroll
          for (int kk = 0; kk < KC / 16; ++kk) {
            const uint64_t bd = sdesc_sw128_mn(v0 + kk * 2048, ATC_SUB, 1024);
            tc_mma_bf16(tO, sdesc_sw128(pa + kk * 32), bd, IDO, (pc > 0 || kk > 0) ? 1u : 0u);
            tc_mma_bf16(tO, sdesc_sw128(pl + kk * 32), bd, IDO, 1u);
            if (SPLIT)  // + Ph.Vl
              tc_mma_bf16(tO, sdesc_sw128(pa + kk * 32), sdesc_sw128_mn(v0 + 4 * ATC_SUB + kk * 2048, ATC_SUB, 1024),
                          IDO, 1u);
          }
          tc_commit(&kempty[pslot]);
          tc_commit(&pvdone);
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax warps 0-3
    const int rl = 16 * warp + (lane & 15), hh = lane >> 4;  // my row, my key half (S) / dim half (O)
    {
      const bf* Qg = reinterpret_cast<const bf*>(P.q);
      for (int i = threadIdx.x; i < QR * 16; i += 128) {
        const int rr = i >> 4, v = i & 15;
        const int slot = sRow[rr];
        const long long qo = (long long)(slot >= 0 ? slot : 0) * D.attn_dim + h * HD + v * 8;
        cp_async16(sQ + (v >> 3) * ATC_SUB + sw128_off(rr, v & 7), Qg + qo, slot >= 0);
        if (SPLIT)
          cp_async16(sQ + 2 * ATC_SUB + (v >> 3) * ATC_SUB + sw128_off(rr, v & 7),
                     reinterpret_cast<const bf*>(P.q_lo) + qo, slot >= 0);
      }
      cp_async_commit();
      cp_async_wait<0>();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&qready);
    }
    const int br_row = sRow[rl] >= 0 ? sBr[rl] : 31;  // bit 31 is never set: no visible key
    const float sl2 = D.attn_scale * 1.4426950408889634f;
    float m_ref = -INFINITY, l_part = 0.0f;
    const uint32_t tl = (uint32_t)(32 * warp) << 16;  // my TMEM lane quadrant
    for (int ci = 0; ci < n_chunks; ++ci) {
      const int slot = ci % NS, sb = ci & 1;
      mbar_wait(&sfull[sb], (ci >> 1) & 1);
      mbar_wait(&kfull[slot], (ci / NS) & 1);  // acquire the producer's visibility words
      tc_fence_after();
      float s[32];
      tmem_ld16x2<32>(tS0 + 64 * sb + tl, s);  // row rl, keys 32*hh + [0, 32)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfree[sb]);
      const uint32_t vw = sVis[slot][br_row][hh];
      float mx4[4] = {m_ref, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        s[c] = ((vw >> c) & 1u) ? s[c] * sl2 : -INFINITY;
        mx4[c & 3] = fmaxf(mx4[c & 3], s[c]);
      }
      float m_new = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
      m_new = fmaxf(m_new, __shfl_xor_sync(0xffffffffu, m_new, 16));
      const bool grow = m_new > m_ref + 8.0f;  // (also the first visible key: m_ref = -inf)
      const float f = !grow ? 1.0f : (m_ref == -INFINITY ? 0.0f : ex2_ftz(m_ref - m_new));
      const float m_old = m_ref;
      if (grow) {
        l_part *= f;
        m_ref = m_new;
      }
      const float mb = m_ref == -INFINITY ? 0.0f : m_ref;
      // P = 2^(s - m) as bf16 hi + lo in registers first: only the stores wait for P(ci-1).V
      uint32_t phi[16], plo[16];
      {
        float ls[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float p0 = ex2_ftz(s[2 * e] - mb), p1 = ex2_ftz(s[2 * e + 1] - mb);
          ls[e & 3] += p0 + p1;
          split_bf2(p0, p1, phi[e], plo[e]);
        }
        l_part += (ls[0] + ls[1]) + (ls[2] + ls[3]);
      }
      // P(ci-1).V done: the P tile is free and O is stable
      if (ci > 0) {
        mbar_wait(&pvdone, (ci - 1) & 1);
        tc_fence_after();
      }
      if (ci > 0 && __any_sync(0xffffffffu, grow && m_old != -INFINITY)) {
        float o[32];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          tmem_ld16x2<64>(tO + tl + 32 * q, o);
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] *= f;
          tmem_st16x2<64>(tO + tl + 32 * q, o);
        }
      }
#pragma unroll
      for (int c8 = 0; c8 < 4; ++c8) {
        const uint32_t off = sw128_off(rl, 4 * hh + c8);
        *reinterpret_cast<uint4*>(sPh + off) = make_uint4(phi[4 * c8], phi[4 * c8 + 1], phi[4 * c8 + 2], phi[4 * c8 + 3]);
        *reinterpret_cast<uint4*>(sPl + off) = make_uint4(plo[4 * c8], plo[4 * c8 + 1], plo[4 * c8 + 2], plo[4 * c8 + 3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pfull);
    }
    if (n_chunks > 0) {
      mbar_wait(&pvdone, (n_chunks - 1) & 1);
      tc_fence_after();
    }
    // partial state (m_ref, l, o / l) of my row half -> fp16 (SPLIT: fp32)
    // staging in the (now idle) KV ring: [QR][HD + 8], (m, l) in the row padding
    constexpr int OLD = HD + 8;
    using ST = typename std::conditional<SPLIT, float, __half>::type;
    ST* sO = reinterpret_cast<ST*>(sKV);
    const float lsum = l_part + __shfl_xor_sync(0xffffffffu, l_part, 16);
    const float il = lsum > 0.0f ? 1.0f / lsum : 0.0f;
    float o[32];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (n_chunks > 0) {
        tmem_ld16x2<64>(tO + tl + 32 * q, o);  // dims 64*hh + 32*q + [0, 32)
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) o[c] = 0.0f;
      }
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        if constexpr (SPLIT)
          *reinterpret_cast<float2*>(sO + rl * OLD + 64 * hh + 32 * q + c) = make_float2(o[c] * il, o[c + 1] * il);
        else
          *reinterpret_cast<__half2*>(sO + rl * OLD + 64 * hh + 32 * q + c) = __floats2half2_rn(o[c] * il, o[c + 1] * il);
      }
    }
    if (hh == 0) *reinterpret_cast<float2*>(sO + rl * OLD + HD) = make_float2(m_ref, lsum);
  }
  tc_fence_before();
  cluster.sync();
  if (threadIdx.x < 128) {
    // merge rows [crank*RPC, (crank+1)*RPC) over the cluster (pull; fixed rank order)
    constexpr int OLD = HD + 8;
    using ST = typename std::conditional<SPLIT, float, __half>::type;
    const ST* sO = reinterpret_cast<const ST*>(sKV);
    constexpr int RPC = QR / CS, V4 = HD / 4, NMI = (RPC * V4 + 127) / 128;
#pragma unroll
    for (int k = 0; k < NMI; ++k) {
      const int i = threadIdx.x + k * 128;
      if (i >= RPC * V4) continue;
      const int lr = crank * RPC + i / V4, c4 = (i % V4) * 4;
      const int slot = sRow[lr];
      float mr[CS], lv[CS];
      float4 ov[CS];
#pragma unroll
      for (int q = 0; q < CS; ++q) {
        const ST* row = cluster.map_shared_rank(sO + lr * OLD, q);
        const float2 ml = *reinterpret_cast<const float2*>(row + HD);
        mr[q] = ml.x;
        lv[q] = ml.y;
        if constexpr (SPLIT) {
          ov[q] = *reinterpret_cast<const float4*>(row + c4);
        } else {
          const uint2 u = *reinterpret_cast<const uint2*>(row + c4);
          const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
          const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
          ov[q] = make_float4(a.x, a.y, b.x, b.y);
        }
      }
      if (slot < 0) continue;
      float M = -INFINITY;
#pragma unroll
      for (int q = 0; q < CS; ++q) M = fmaxf(M, mr[q]);
      float Lsum = 0.0f;
      float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
      for (int q = 0; q < CS; ++q) {
        if (mr[q] == -INFINITY || lv[q] <= 0.0f) continue;
        const float w = ex2_ftz(mr[q] - M) * lv[q];
        Lsum += w;
        acc.x += w * ov[q].x;
        acc.y += w * ov[q].y;
        acc.z += w * ov[q].z;
        acc.w += w * ov[q].w;
      }
      const float inv = Lsum > 0.0f ? 1.0f / Lsum : 0.0f;
      const long long oo = (long long)slot * D.attn_dim + h * HD + c4;
      const float4 y = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
      __nv_bfloat162 p0 = __floats2bfloat162_rn(y.x, y.y), p1 = __floats2bfloat162_rn(y.z, y.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&p0);
      u.y = *reinterpret_cast<uint32_t*>(&p1);
      *reinterpret_cast<uint2*>(reinterpret_cast<bf*>(P.attn) + oo) = u;
      if (SPLIT) {  // lo = rn(y - hi)
        const float2 f0 = __bfloat1622float2(p0), f1 = __bfloat1622float2(p1);
        __nv_bfloat162 l0 = __floats2bfloat162_rn(y.x - f0.x, y.y - f0.y), l1 = __floats2bfloat162_rn(y.z - f1.x, y.w - f1.y);
        u.x = *reinterpret_cast<uint32_t*>(&l0);
        u.y = *reinterpret_cast<uint32_t*>(&l1);
        *reinterpret_cast<uint2*>(reinterpret_cast<bf*>(P.attn_lo) + oo) = u;
      }
    }
  }
  cluster.sync();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(s_tmem, 256);
  }
  tstat_end(ats);
}

template <int NS, bool SPLIT>
constexpr size_t attn_fa_smem() {
  return 1024 + (size_t)((SPLIT ? 2 : 1) * (2 + 4 * NS) + 2) * ATC_SUB;  // q, KV ring, P hi + lo
}

template <int CS, int NS, bool SPLIT>
static cudaError_t attn_fa_launch(const Dims& D, const Sess& S, const Pass& P, const DevState& st,
                                  const AttnMaps& am, int layer, cudaStream_t s) {
  const int rows = P.full ? S.L : S.NRq;
  constexpr size_t smem = attn_fa_smem<NS, SPLIT>();
  static_assert(smem <= 227 * 1024, "k_attn_fa shared memory");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_attn_fa<CS, NS, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid(pass_groups(S, P) * CS, D.nh, (rows + ATC_QR - 1) / ATC_QR);
  launch_k(k_attn_fa<CS, NS, SPLIT>, dim3(grid), dim3(AFA_THREADS), smem, s, am.k, am.v, am.kl, am.vl, D, S, P, st,
           layer, rows);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ M = 128 warp-specialized attention
// k_attn_fa128: k_attn_fa's roles and pipeline on 128-row query tiles (one
// tcgen05 M=128 accumulator: TMEM lane = query row, so each softmax thread
// owns one whole row -- no lane pairs, no shuffles), half the MMA
// instructions per row of the M=64 kernel, and a key tile's K/V pages read
// once for up to 128 rows (every branch window of a C2 / C5 block pass).
//   smem: q 32 KB | NS x (K 16 KB + V 16 KB) | NPB x P (hi 16 KB + lo 16 KB)
//   TMEM: S0, S1 (64 columns each), O (128 columns)
// SPLIT (bf16x2): q / K / V hi + lo planes (the products of k_attn_fa's SPLIT
// instance), fp32 cluster merge, hi + lo output; q 64 KB + 2 x 64 KB stages +
// one P buffer = the whole opt-in shared memory.
constexpr int AF8_QR = 128;
constexpr uint32_t AF8_SUB = 128 * 128;  // one [128 rows][64 bf16] SW128 sub-tile (bytes)

template <int CS, int NS, bool SPLIT>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(AFA_THREADS)
    k_attn_fa128(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                 const __grid_constant__ CUtensorMap tmKl, const __grid_constant__ CUtensorMap tmVl, Dims D, Sess S,
                 Pass P, DevState st, int layer, int rows_per_req) {
  klog_mark(D.klog, D.klog_cap, 24);
  if (P.pf_base != nullptr && threadIdx.x == 0) {
    // this CTA's slice of the O projection's weights -> L2 (HBM is not saturated by the attention)
    const long long n_cta = (long long)gridDim.x * gridDim.y * gridDim.z;
    const long long cta = blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
    const long long per = ((P.pf_layer_bytes + n_cta - 1) / n_cta + 127) & ~127LL;
    const char* base = P.pf_base + (long long)layer * P.pf_layer_bytes;
    for (long long o = cta * per; o < min((cta + 1) * per, P.pf_layer_bytes); o += 65536) {
      const long long n = min(65536LL, min((cta + 1) * per, P.pf_layer_bytes) - o);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"((uint32_t)n) : "memory");
    }
  }
  using bf = __nv_bfloat16;
  constexpr int HD = ATC_HD, QR = AF8_QR, KC = ATC_KC;
  constexpr int NP = SPLIT ? 2 : 1;              // hi (+ lo) planes
  constexpr int NPB = SPLIT ? 1 : 2;             // P buffers
  constexpr uint32_t STAGE = NP * 4 * ATC_SUB;   // [K hi 2 sub, V hi 2 sub (, K lo 2, V lo 2)], sub = [64 keys][64 dims]
  extern __shared__ __align__(1024) uint8_t smraw_f8[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw_f8) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;                      // [plane][2 sub-tiles [128 rows][64 dims]]
  uint8_t* sKV = sQ + NP * 2 * AF8_SUB;  // [NS] stages
  uint8_t* sP = sKV + NS * STAGE;   // [2 buffers][hi, lo][128 rows][64 keys] K-major
  __shared__ int sRow[QR], sBr[QR];
  __shared__ uint32_t sVis[NS][32][2];  // [slot][branch][key word]
  __shared__ int s_nk;
  // P is double-buffered (chunk c in buffer c & 1, hand-offs on pfull / pvdone[c & 1]): the
  // softmax of chunk ci waits only for P(ci-2).V (long done) -- or P(ci-1).V when O must be rescaled
  __shared__ __align__(8) uint64_t kfull[NS], kempty[NS], sfull[2], sfree[2], pfull[2], pvdone[2], qready;
  __shared__ uint32_t s_tmem;

  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int r = blockIdx.x / CS, h = blockIdx.y;
  const int row0 = blockIdx.z * QR;
  const int kvh = h / (D.nh / D.nkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int slot_base = -1;  // block pass: read after the dependency wait (compacting sessions rewrite it)
  const long long kb = (long long)r * P.n_kz + (P.full ? 0 : ((blockIdx.z * QR) >> P.kz_shift));

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kfull[i], 1);
      mbar_init(&kempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sfree[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&pfull[i], 4);
      mbar_init(&pvdone[i], 1);
    }
    mbar_init(&qready, 128);
    fence_mbar_init();
  }
  if (warp == 4 && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    if (SPLIT) {
      tma_prefetch_desc(&tmKl);
      tma_prefetch_desc(&tmVl);
    }
  }
  if (warp == 5) tmem_alloc(&s_tmem, 256);  // S0, S1: 64 columns each; O: 128 columns
  pdl_enter();
  slot_base = P.full ? r * S.L : blk_base(S, P, r);  // -1: finished request (compacting session)
  klog_mark(D.klog, D.klog_cap, 3);
  unsigned long long* const ats = D.klog != nullptr ? P.atstat : nullptr;
  tstat_begin(ats);
  if (threadIdx.x < QR) {
    const int lr = row0 + threadIdx.x;
    int slot = -1, br = 0;
    if (lr < rows_per_req && slot_base >= 0) {
      const int sl = slot_base + lr;
      br = P.slot_br[sl];
      if (P.slot_pos[sl] >= 0 && !*P.skip) slot = sl;
    }
    sRow[threadIdx.x] = slot;
    sBr[threadIdx.x] = br;
  } else if (threadIdx.x == QR) {
    s_nk = P.akey_n[2 * kb];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tS0 = s_tmem, tO = s_tmem + 128;
  const int n_keys = s_nk;
  const int nc_all = (n_keys + KC - 1) / KC;
  const int c_begin = (int)((long long)nc_all * crank / CS);
  const int n_chunks = (int)((long long)nc_all * (crank + 1) / CS) - c_begin;
  const int k_begin = c_begin * KC;
  const int2* ksrc = reinterpret_cast<const int2*>(P.akeys) + kb * P.akey_cap + k_begin;
  const int nk_cta = min(n_keys - k_begin, n_chunks * KC);

  if (warp == 4) {
    // ---------------- producer (as k_attn_fa)
    const uint64_t pol = policy_evict_normal();
    const int lay_rows = layer * S.R * S.pool;
    auto entries = [&](int ci, int2& e0, int2& e1) {
      const int i0 = ci * KC + lane, i1 = i0 + 32;
      e0 = (ci < n_chunks && i0 < nk_cta) ? ksrc[i0] : make_int2(0, 0);
      e1 = (ci < n_chunks && i1 < nk_cta) ? ksrc[i1] : make_int2(0, 0);
    };
    int2 e0, e1, n0, n1;
    entries(0, e0, e1);
    for (int ci = 0; ci < n_chunks; ++ci) {
      const int slot = ci % NS;
      uint32_t vis[2 * MAXB];
#pragma unroll
      for (int b = 0; b < MAXB; ++b) {
        vis[2 * b] = __ballot_sync(0xffffffffu, b < S.B && ((e0.y >> b) & 1));
        vis[2 * b + 1] = __ballot_sync(0xffffffffu, b < S.B && ((e1.y >> b) & 1));
      }
      const int pg0 = __shfl_sync(0xffffffffu, e0.x, 0) >> 4, pg1 = __shfl_sync(0xffffffffu, e0.x, 16) >> 4;
      const int pg2 = __shfl_sync(0xffffffffu, e1.x, 0) >> 4, pg3 = __shfl_sync(0xffffffffu, e1.x, 16) >> 4;
      entries(ci + 1, n0, n1);
      if (ci >= NS) mbar_wait(&kempty[slot], ((ci / NS) - 1) & 1);
      if (lane == 0) {
#pragma unroll
        for (int b = 0; b < MAXB; ++b) {
          sVis[slot][b][0] = vis[2 * b];
          sVis[slot][b][1] = vis[2 * b + 1];
        }
        sVis[slot][31][0] = 0u;
        sVis[slot][31][1] = 0u;
        const int nk = min(KC, nk_cta - ci * KC);
        const int pgs[4] = {pg0, nk > 16 ? pg1 : pg0, nk > 32 ? pg2 : pg0, nk > 48 ? pg3 : pg0};
        uint8_t* dst = sKV + slot * STAGE;
        mbar_expect_tx(&kfull[slot], STAGE);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int row = ((lay_rows + pgs[g]) * D.nkv + kvh) * 16;
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {
            tma_load_2d(dst + sub * ATC_SUB + g * 2048, &tmK, &kfull[slot], sub * 64, row, pol);
            tma_load_2d(dst + (2 + sub) * ATC_SUB + g * 2048, &tmV, &kfull[slot], sub * 64, row, pol);
            if (SPLIT) {
              tma_load_2d(dst + (4 + sub) * ATC_SUB + g * 2048, &tmKl, &kfull[slot], sub * 64, row, pol);
              tma_load_2d(dst + (6 + sub) * ATC_SUB + g * 2048, &tmVl, &kfull[slot], sub * 64, row, pol);
            }
          }
        }
      }
      e0 = n0;
      e1 = n1;
      __syncwarp();
    }
  } else if (warp == 5) {
    // ---------------- MMA issuer (readiness order)
    if (lane == 0 && n_chunks > 0) {
      constexpr uint32_t IDS = idesc_bf16_f32(128, 64);
      constexpr uint32_t IDO = idesc_bf16_f32(128, 128) | (1u << 16);  // B (V) MN-major
      mbar_wait(&qready, 0);
      tc_fence_after();
      const uint32_t q0 = smem_u32(sQ);
      // issue order.  One P buffer (SPLIT): by readiness -- S(ci) as soon as its chunk
      // landed and its S buffer was read, P(cp).V as soon as P(cp) is written (S first
      // when both are), so a P.V never waits behind the next chunk's load (C5 block
      // attention 150 -> 120 us).  Two P buffers: S(ci) then P(ci-1).V, strictly
      // (readiness order measured 2% slower there).
      constexpr bool RDY = NPB == 1;
      int ci = 0, cp = 0;
      const long long t_spin = clock64();
      while (cp < n_chunks) {
        bool s_ok = false;
        if (ci < n_chunks && (RDY || cp >= ci - 1)) {
          const int slot = ci % NS, sb = ci & 1;
          s_ok = mbar_try_wait(smem_u32(&kfull[slot]), (ci / NS) & 1) &&
                 (ci < 2 || mbar_try_wait(smem_u32(&sfree[sb]), ((ci >> 1) - 1) & 1));
        }
        if (s_ok) {
          const int slot = ci % NS, sb = ci & 1;
          tc_fence_after();
          const uint32_t k0 = smem_u32(sKV + slot * STAGE);
#pragma unroll
          for (int ks = 0; ks < HD / 16; ++ks) {
            const uint32_t ko = (ks & 3) * 32;
            tc_mma_bf16(tS0 + 64 * sb, sdesc_sw128(q0 + (ks >> 2) * AF8_SUB + ko),
                        sdesc_sw128(k0 + (ks >> 2) * ATC_SUB + ko), IDS, ks > 0 ? 1u : 0u);
          }
          if (SPLIT) {  // + Qh.Kl + Ql.Kh
            const uint32_t ql = q0 + 2 * AF8_SUB, kl = k0 + 4 * ATC_SUB;
#pragma unroll
            for (int ks = 0; ks < HD / 16; ++ks) {
              const uint32_t ko = (ks & 3) * 32;
              tc_mma_bf16(tS0 + 64 * sb, sdesc_sw128(q0 + (ks >> 2) * AF8_SUB + ko),
                          sdesc_sw128(kl + (ks >> 2) * ATC_SUB + ko), IDS, 1u);
              tc_mma_bf16(tS0 + 64 * sb, sdesc_sw128(ql + (ks >> 2) * AF8_SUB + ko),
                          sdesc_sw128(k0 + (ks >> 2) * ATC_SUB + ko), IDS, 1u);
            }
          }
          tc_commit(&sfull[sb]);
          ++ci;
        } else if (cp < ci && (RDY || ci >= min(cp + 2, n_chunks)) &&
                   mbar_try_wait(smem_u32(&pfull[cp % NPB]), (cp / NPB) & 1)) {
          const int pc = cp, pslot = pc % NS, pb = pc % NPB;
          tc_fence_after();
          const uint32_t v0 = smem_u32(sKV + pslot * STAGE + 2 * ATC_SUB);
          const uint32_t pa = smem_u32(sP + pb * 2 * AF8_SUB), pl = pa + AF8_SUB;
#pragma unroll
          for (int kk = 0; kk < KC / 16; ++kk) {
            const uint64_t bd = sdesc_sw128_mn(v0 + kk * 2048, ATC_SUB, 1024);
            tc_mma_bf16(tO, sdesc_sw128(pa + kk * 32), bd, IDO, (pc > 0 || kk > 0) ? 1u : 0u);
            tc_mma_bf16(tO, sdesc_sw128(pl + kk * 32), bd, IDO, 1u);
            if (SPLIT)  // + Ph.Vl
              tc_mma_bf16(tO, sdesc_sw128(pa + kk * 32), sdesc_sw128_mn(v0 + 4 * ATC_SUB + kk * 2048, ATC_SUB, 1024),
                          IDO, 1u);
          }
          tc_commit(&kempty[pslot]);
          tc_commit(&pvdone[pb]);
          ++cp;
        } else if (clock64() - t_spin > (long long)20000000000LL) {
          __trap();
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax warps 0-3: thread t owns query row t (TMEM lane t)
    const int rl = threadIdx.x;
    {
      const bf* Qg = reinterpret_cast<const bf*>(P.q);
      for (int i = threadIdx.x; i < QR * 16; i += 128) {
        const int rr = i >> 4, v = i & 15;
        const int slot = sRow[rr];
        const long long qo = (long long)(slot >= 0 ? slot : 0) * D.attn_dim + h * HD + v * 8;
        cp_async16(sQ + (v >> 3) * AF8_SUB + sw128_off(rr, v & 7), Qg + qo, slot >= 0);
        if (SPLIT)
          cp_async16(sQ + 2 * AF8_SUB + (v >> 3) * AF8_SUB + sw128_off(rr, v & 7),
                     reinterpret_cast<const bf*>(P.q_lo) + qo, slot >= 0);
      }
      cp_async_commit();
      cp_async_wait<0>();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&qready);
    }
    const int br_row = sRow[rl] >= 0 ? sBr[rl] : 31;  // bit 31 is never set: no visible key
    const float sl2 = D.attn_scale * 1.4426950408889634f;
    float m_ref = -INFINITY, l_part = 0.0f;
    const uint32_t tl = (uint32_t)(32 * warp) << 16;  // my TMEM lane quadrant
    for (int ci = 0; ci < n_chunks; ++ci) {
      const int slot = ci % NS, sb = ci & 1;
      mbar_wait(&sfull[sb], (ci >> 1) & 1);
      mbar_wait(&kfull[slot], (ci / NS) & 1);  // acquire the producer's visibility words
      tc_fence_after();
      float s[64];
      {
        float a[32], b[32];
        tmem_ld32(tS0 + 64 * sb + tl, a);
        tmem_ld32(tS0 + 64 * sb + tl + 32, b);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          s[c] = a[c];
          s[32 + c] = b[c];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfree[sb]);
      const uint32_t v0 = sVis[slot][br_row][0], v1 = sVis[slot][br_row][1];
      float mx4[4] = {m_ref, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 64; ++c) {
        const uint32_t vw = c < 32 ? v0 : v1;
        s[c] = ((vw >> (c & 31)) & 1u) ? s[c] * sl2 : -INFINITY;
        mx4[c & 3] = fmaxf(mx4[c & 3], s[c]);
      }
      const float m_new = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
      const bool grow = m_new > m_ref + 8.0f;  // (also the first visible key: m_ref = -inf)
      const float f = !grow ? 1.0f : (m_ref == -INFINITY ? 0.0f : ex2_ftz(m_ref - m_new));
      const float m_old = m_ref;
      if (grow) {
        l_part *= f;
        m_ref = m_new;
      }
      const float mb = m_ref == -INFINITY ? 0.0f : m_ref;
      {
        float ls[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          s[c] = ex2_ftz(s[c] - mb);
          ls[c & 3] += s[c];
        }
        l_part += (ls[0] + ls[1]) + (ls[2] + ls[3]);
      }
      // P buffer free (two buffers: P(ci-2).V done; one: P(ci-1).V done); a rescale also
      // needs O stable: P(ci-1).V done
      const int pb = ci % NPB;
      const bool rescale = ci > 0 && __any_sync(0xffffffffu, grow && m_old != -INFINITY);
      if (NPB == 2) {
        if (ci >= 2) mbar_wait(&pvdone[pb], ((ci - 2) >> 1) & 1);
        if (rescale) mbar_wait(&pvdone[pb ^ 1], ((ci - 1) >> 1) & 1);
      } else if (ci >= 1) {
        mbar_wait(&pvdone[0], (ci - 1) & 1);
      }
      if (ci >= 1) tc_fence_after();
      if (rescale) {
        float o[32];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          tmem_ld32(tO + tl + 32 * q, o);
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] *= f;
          tmem_st32(tO + tl + 32 * q, o);
        }
      }
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) {
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split_bf2(s[8 * c8 + 2 * e], s[8 * c8 + 2 * e + 1], hi[e], lo[e]);
        const uint32_t off = sw128_off(rl, c8);
        *reinterpret_cast<uint4*>(sP + pb * 2 * AF8_SUB + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(sP + (pb * 2 + 1) * AF8_SUB + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pfull[pb]);
    }
    if (n_chunks > 0) {  // the last P.V (its commit also covers every earlier one)
      mbar_wait(&pvdone[(n_chunks - 1) % NPB], ((n_chunks - 1) / NPB) & 1);
      tc_fence_after();
    }
    // partial state (m_ref, l, o / l) of my row -> fp16 (SPLIT: fp32) staging in the idle KV ring
    constexpr int OLD = HD + 8;
    using ST = typename std::conditional<SPLIT, float, __half>::type;
    ST* sO = reinterpret_cast<ST*>(sKV);
    const float il = l_part > 0.0f ? 1.0f / l_part : 0.0f;
    float o[32];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (n_chunks > 0) {
        tmem_ld32(tO + tl + 32 * q, o);
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) o[c] = 0.0f;
      }
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        if constexpr (SPLIT)
          *reinterpret_cast<float2*>(sO + rl * OLD + 32 * q + c) = make_float2(o[c] * il, o[c + 1] * il);
        else
          *reinterpret_cast<__half2*>(sO + rl * OLD + 32 * q + c) = __floats2half2_rn(o[c] * il, o[c + 1] * il);
      }
    }
    *reinterpret_cast<float2*>(sO + rl * OLD + HD) = make_float2(m_ref, l_part);
  }
  tc_fence_before();
  cluster.sync();
  if (threadIdx.x < 128) {
    // merge rows [crank*RPC, (crank+1)*RPC) over the cluster (pull; fixed rank order)
    constexpr int OLD = HD + 8;
    using ST = typename std::conditional<SPLIT, float, __half>::type;
    const ST* sO = reinterpret_cast<const ST*>(sKV);
    constexpr int RPC = QR / CS, V4 = HD / 4, NMI = (RPC * V4 + 127) / 128;
#pragma unroll
    for (int k = 0; k < NMI; ++k) {
      const int i = threadIdx.x + k * 128;
      if (i >= RPC * V4) continue;
      const int lr = crank * RPC + i / V4, c4 = (i % V4) * 4;
      const int slot = sRow[lr];
      if (slot < 0) continue;
      float mr[CS], lv[CS];
      float4 ov[CS];
#pragma unroll
      for (int q = 0; q < CS; ++q) {
        const ST* row = cluster.map_shared_rank(sO + lr * OLD, q);
        const float2 ml = *reinterpret_cast<const float2*>(row + HD);
        mr[q] = ml.x;
        lv[q] = ml.y;
        if constexpr (SPLIT) {
          ov[q] = *reinterpret_cast<const float4*>(row + c4);
        } else {
          const uint2 u = *reinterpret_cast<const uint2*>(row + c4);
          const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
          const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
          ov[q] = make_float4(a.x, a.y, b.x, b.y);
        }
      }
      float M = -INFINITY;
#pragma unroll
      for (int q = 0; q < CS; ++q) M = fmaxf(M, mr[q]);
      float Lsum = 0.0f;
      float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
      for (int q = 0; q < CS; ++q) {
        if (mr[q] == -INFINITY || lv[q] <= 0.0f) continue;
        const float w = ex2_ftz(mr[q] - M) * lv[q];
        Lsum += w;
        acc.x += w * ov[q].x;
        acc.y += w * ov[q].y;
        acc.z += w * ov[q].z;
        acc.w += w * ov[q].w;
      }
      const float inv = Lsum > 0.0f ? 1.0f / Lsum : 0.0f;
      const long long oo = (long long)slot * D.attn_dim + h * HD + c4;
      const float4 y = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
      __nv_bfloat162 p0 = __floats2bfloat162_rn(y.x, y.y), p1 = __floats2bfloat162_rn(y.z, y.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&p0);
      u.y = *reinterpret_cast<uint32_t*>(&p1);
      *reinterpret_cast<uint2*>(reinterpret_cast<bf*>(P.attn) + oo) = u;
      if (SPLIT) {  // lo = rn(y - hi)
        const float2 f0 = __bfloat1622float2(p0), f1 = __bfloat1622float2(p1);
        __nv_bfloat162 l0 = __floats2bfloat162_rn(y.x - f0.x, y.y - f0.y), l1 = __floats2bfloat162_rn(y.z - f1.x, y.w - f1.y);
        u.x = *reinterpret_cast<uint32_t*>(&l0);
        u.y = *reinterpret_cast<uint32_t*>(&l1);
        *reinterpret_cast<uint2*>(reinterpret_cast<bf*>(P.attn_lo) + oo) = u;
      }
    }
  }
  cluster.sync();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(s_tmem, 256);
  }
  tstat_end(ats);
}

template <int NS, bool SPLIT>
constexpr size_t attn_f8_smem() {
  // q (hi (+ lo)) + P buffers (2 plain, 1 SPLIT; hi + lo each) + the KV ring
  return 1024 + (size_t)(SPLIT ? 4 + 2 : 2 + 4) * AF8_SUB + (size_t)NS * (SPLIT ? 8 : 4) * ATC_SUB;
}

template <int CS, int NS, bool SPLIT>
static long long f8_slots() {
  static long long v = -1;
  if (v < 0) {
    constexpr size_t smem = attn_f8_smem<NS, SPLIT>();
    cudaFuncSetAttribute(k_attn_fa128<CS, NS, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS * 64);
    cfg.blockDim = dim3(AFA_THREADS);
    cfg.dynamicSmemBytes = smem;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (void*)k_attn_fa128<CS, NS, SPLIT>, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148 / CS;
    }
    v = (long long)n * CS;
    if (getenv("BB_DEBUG"))
      fprintf(stderr, "[bb200] k_attn_fa128<%d,%d,%d>: %d resident clusters\n", CS, NS, (int)SPLIT, n);
  }
  return v;
}

template <int CS, int NS, bool SPLIT>
static cudaError_t attn_f8_launch(const Dims& D, const Sess& S, const Pass& P, const DevState& st,
                                  const AttnMaps& am, int layer, cudaStream_t s) {
  const int rows = P.full ? S.L : S.NRq;
  constexpr size_t smem = attn_f8_smem<NS, SPLIT>();
  static_assert(smem + 2048 <= 232448, "k_attn_fa128 shared memory (dynamic + static)");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_attn_fa128<CS, NS, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid(pass_groups(S, P) * CS, D.nh, (rows + AF8_QR - 1) / AF8_QR);
  launch_k(k_attn_fa128<CS, NS, SPLIT>, dim3(grid), dim3(AFA_THREADS), smem, s, am.k, am.v, am.kl, am.vl, D, S, P, st,
           layer, rows);
  return cudaGetLastError();
}

#ifndef ATT_F8_NS
#define ATT_F8_NS 3  // KV ring stages of k_attn_fa128 (one CTA per SM); the SPLIT instance has 2
#endif
template <int NS, bool SPLIT>
static int att_cs_f8(const Dims& D, const Sess& S, const Pass& P, int tflags) {
  const int forced = (tflags >> 4) & 15;
  if (forced == 8 || forced == 4 || forced == 2 || forced == 1) return forced;
  const int rows = P.full ? S.L : S.NRq;
  const long long per = (long long)pass_groups(S, P) * D.nh * ((rows + AF8_QR - 1) / AF8_QR);
  if (per * 8 <= 2 * f8_slots<8, NS, SPLIT>()) return 8;
  if (per * 4 <= 2 * f8_slots<4, NS, SPLIT>()) return 4;
  if (per * 2 <= 2 * f8_slots<2, NS, SPLIT>()) return 2;
  return 1;
}

// tcgen05 attention for hd = 128 in every pass (block, prefill, refresh).
// Measured (C5 block attention 222 vs 262 us per launch for the mma.sync
// kernel, C5 16.7 vs 17.9 ms/NFE; C2 attention slot 16.8 vs 19.4 us).
// Cluster size for k_attn_tc (2 CTAs/SM): the largest of 8 / 4 / 2 / 1 whose
// grid fits one wave, else 1 (splitting keys over a cluster only pays while
// the (request, head, row tile) units alone cannot fill the GPU).  C5 full
// passes (1536 units): CS 8 / 4 / 2 = 1020 / 829 / 731 us per launch.
static int att_cs_tc(const Dims& D, const Sess& S, const Pass& P, int tflags, int per_sm) {
  const int forced = (tflags >> 4) & 15;
  if (forced == 8 || forced == 4 || forced == 2 || forced == 1) return forced;
  const int rows = P.full ? S.L : S.NRq;
  const long long per = (long long)pass_groups(S, P) * D.nh * ((rows + ATC_QR - 1) / ATC_QR);
  const long long wave = (long long)per_sm * S.n_sms;  // resident CTAs per SM x SMs
  for (int cs = 8; cs > 1; cs >>= 1)
    if (per * cs <= wave) return cs;
  return 1;
}

// test flag bit 0 (BB_TF_ATTN_MMA_SYNC): the mma.sync kernel at hd 128 (tests
// compare the two tensor-core attentions; never set on the product path)
#ifndef ATT_FA_NS
#define ATT_FA_NS 2  // KV ring stages of k_attn_fa (2: 99 KB, two CTAs per SM)
#endif
// Resident CTAs of k_attn_fa<CS> in clusters (occupancy API, cached): the
// cluster placement, not smem alone, bounds how many fit at once.
template <int CS, int NS, bool SPLIT>
static long long fa_slots() {
  static long long v = -1;
  if (v < 0) {
    constexpr size_t smem = attn_fa_smem<NS, SPLIT>();
    cudaFuncSetAttribute(k_attn_fa<CS, NS, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS * 64);
    cfg.blockDim = dim3(AFA_THREADS);
    cfg.dynamicSmemBytes = smem;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (void*)k_attn_fa<CS, NS, SPLIT>, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148 / CS;
    }
    v = (long long)n * CS;
    if (getenv("BB_DEBUG")) fprintf(stderr, "[bb200] k_attn_fa<%d,%d,%d>: %d resident clusters\n", CS, NS, (int)SPLIT, n);
  }
  return v;
}
// Cluster size of k_attn_fa: the largest CS whose grid runs in at most two
// waves.  The chunk loop runs at a per-SM rate, so splitting a (request,
// head, row tile)'s keys finer mainly evens out the SMs' loads (row tiles
// see different key counts); measured C5 block pass CS 1/2/4/8 = 321 / 173
// / 91 / 76 us, C5 full pass 651 / 641 / 715 / 886 us (1536 units).
template <int NS, bool SPLIT>
static int att_cs_fa(const Dims& D, const Sess& S, const Pass& P, int tflags) {
  const int forced = (tflags >> 4) & 15;
  if (forced == 8 || forced == 4 || forced == 2 || forced == 1) return forced;
  const int rows = P.full ? S.L : S.NRq;
  const long long per = (long long)pass_groups(S, P) * D.nh * ((rows + ATC_QR - 1) / ATC_QR);
  if (per * 8 <= 2 * fa_slots<8, NS, SPLIT>()) return 8;
  if (per * 4 <= 2 * fa_slots<4, NS, SPLIT>()) return 4;
  if (per * 2 <= 2 * fa_slots<2, NS, SPLIT>()) return 2;
  return 1;
}
template <int HD>
static cudaError_t attn_seg_hd(const Dims& D, const Sess& S, const Pass& P, const DevState& st, const AttnMaps& am,
                               int layer, int tflags, cudaStream_t s) {
  if constexpr (HD == 128) {
    // product path: the warp-specialized TMA-fed kernels -- M = 128 row tiles
    // (bf16), M = 64 (bf16x2, whose q / KV planes double the shared memory);
    // test flag bit 1 = k_attn_tc, bit 2 = the M = 64 kernel for bf16
    if (am.ok && !(tflags & 3) && P.kz_shift == 7) {
      if (D.split) {
        switch (att_cs_f8<2, true>(D, S, P, tflags)) {
          case 8: return attn_f8_launch<8, 2, true>(D, S, P, st, am, layer, s);
          case 4: return attn_f8_launch<4, 2, true>(D, S, P, st, am, layer, s);
          case 2: return attn_f8_launch<2, 2, true>(D, S, P, st, am, layer, s);
          default: return attn_f8_launch<1, 2, true>(D, S, P, st, am, layer, s);
        }
      }
      switch (att_cs_f8<ATT_F8_NS, false>(D, S, P, tflags)) {
        case 8: return attn_f8_launch<8, ATT_F8_NS, false>(D, S, P, st, am, layer, s);
        case 4: return attn_f8_launch<4, ATT_F8_NS, false>(D, S, P, st, am, layer, s);
        case 2: return attn_f8_launch<2, ATT_F8_NS, false>(D, S, P, st, am, layer, s);
        default: return attn_f8_launch<1, ATT_F8_NS, false>(D, S, P, st, am, layer, s);
      }
    }
    if (am.ok && !(tflags & 3)) {
      if (D.split) {
        switch (att_cs_fa<2, true>(D, S, P, tflags)) {
          case 8: return attn_fa_launch<8, 2, true>(D, S, P, st, am, layer, s);
          case 4: return attn_fa_launch<4, 2, true>(D, S, P, st, am, layer, s);
          case 2: return attn_fa_launch<2, 2, true>(D, S, P, st, am, layer, s);
          default: return attn_fa_launch<1, 2, true>(D, S, P, st, am, layer, s);
        }
      }
      switch (att_cs_fa<ATT_FA_NS, false>(D, S, P, tflags)) {
        case 8: return attn_fa_launch<8, ATT_FA_NS, false>(D, S, P, st, am, layer, s);
        case 4: return attn_fa_launch<4, ATT_FA_NS, false>(D, S, P, st, am, layer, s);
        case 2: return attn_fa_launch<2, ATT_FA_NS, false>(D, S, P, st, am, layer, s);
        default: return attn_fa_launch<1, ATT_FA_NS, false>(D, S, P, st, am, layer, s);
      }
    }
    if (D.split) {  // bf16x2: the tcgen05 attention only
      switch (att_cs_tc(D, S, P, tflags, 1)) {
        case 8: return attn_tc_launch<8, true>(D, S, P, st, layer, s);
        case 4: return attn_tc_launch<4, true>(D, S, P, st, layer, s);
        case 2: return attn_tc_launch<2, true>(D, S, P, st, layer, s);
        default: return attn_tc_launch<1, true>(D, S, P, st, layer, s);
      }
    }
    if (!(tflags & 1)) {
      switch (att_cs_tc(D, S, P, tflags, 2)) {
        case 8: return attn_tc_launch<8, false>(D, S, P, st, layer, s);
        case 4: return attn_tc_launch<4, false>(D, S, P, st, layer, s);
        case 2: return attn_tc_launch<2, false>(D, S, P, st, layer, s);
        default: return attn_tc_launch<1, false>(D, S, P, st, layer, s);
      }
    }
  }
  switch (att_cs(D, S, P, tflags)) {
    case 8: return attn_seg_launch<HD, 8>(D, S, P, st, layer, s);
    case 4: return attn_seg_launch<HD, 4>(D, S, P, st, layer, s);
    case 2: return attn_seg_launch<HD, 2>(D, S, P, st, layer, s);
    default: return attn_seg_launch<HD, 1>(D, S, P, st, layer, s);
  }
}

// LSE-merge of the partials of the items covering (row, head).  CTA per
// (row, head), one thread per head dim; fixed item order (deterministic).
template <typename T>
__global__ void __launch_bounds__(256) k_attn_combine2(Dims D, Sess S, Pass P, int max_items) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 22);
  if (*P.skip) return;
  const int row = blockIdx.x, h = blockIdx.y;
  const int pos = P.slot_pos[row];
  if (pos < 0) return;
  const int r = P.slot_req[row], k = P.slot_br[row];
  const int j = row - P.rng_off[r * MAXB + k];
  if (j < 0 || j >= P.rng_cnt[r * MAXB + k]) return;
  __shared__ int s_off[256];
  __shared__ int s_n;
  const int HD = D.hd;
  // parallel scan of the request's items: which cover this row's branch, at which item row
  const int ni = P.n_items[r];
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  for (int base = 0; base < ni; base += blockDim.x) {
    const int it = base + threadIdx.x;
    int cover = 0, off = 0;
    if (it < ni) {
      const int mask = P.items[((long long)r * max_items + it) * ITW];
      if ((mask >> k) & 1) {
        int rii = j;
        for (int k2 = 0; k2 < k; ++k2)
          if ((mask >> k2) & 1) rii += P.rng_cnt[r * MAXB + k2];
        cover = 1;
        off = (int)((((long long)r * max_items + it) * P.item_rows + rii) * D.nh + h);
      }
    }
    // stable compaction (item order preserved -> deterministic merge order)
    const unsigned ballot = __ballot_sync(0xffffffffu, cover);
    __shared__ int s_wc[8];
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    if (ln == 0) s_wc[w] = __popc(ballot);
    __syncthreads();
    int pre = s_n;
    for (int ww = 0; ww < w; ++ww) pre += s_wc[ww];
    pre += __popc(ballot & ((1u << ln) - 1u));
    if (cover && pre < 256) s_off[pre] = off;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) tot += s_wc[ww];
      s_n = min(256, s_n + tot);
    }
    __syncthreads();
  }
  const int n = s_n;
  float M = -INFINITY;
  for (int i = 0; i < n; ++i) M = fmaxf(M, P.apart[(long long)s_off[i] * (HD + 2) + HD]);
  T* out = reinterpret_cast<T*>(P.attn) + (long long)row * D.attn_dim + h * HD;
  for (int c = threadIdx.x; c < HD; c += blockDim.x) {
    float acc = 0.0f, L = 0.0f;
    for (int i = 0; i < n; ++i) {
      const float* o = P.apart + (long long)s_off[i] * (HD + 2);
      const float mi = o[HD];
      if (mi == -INFINITY) continue;
      const float w = expf(mi - M);
      acc = fmaf(o[c], w, acc);
      L = fmaf(o[HD + 1], w, L);
    }
    stf(out + c, acc / L);
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
  launch_k(k_attn<T, HD>, dim3(grid), dim3(128), (size_t)(smem), s, D, S, P, st, layer, max_items);
  return cudaGetLastError();
}


// Occupancy queries of the k_attn_fa instances (cluster residency), run at
// session creation: they are not allowed inside a stream capture.
void attn_prepare() {
  f8_slots<8, ATT_F8_NS, false>();
  f8_slots<4, ATT_F8_NS, false>();
  f8_slots<2, ATT_F8_NS, false>();
  f8_slots<8, 2, true>();
  f8_slots<4, 2, true>();
  f8_slots<2, 2, true>();
  fa_slots<8, ATT_FA_NS, false>();
  fa_slots<4, ATT_FA_NS, false>();
  fa_slots<2, ATT_FA_NS, false>();
  fa_slots<8, 2, true>();
  fa_slots<4, 2, true>();
  fa_slots<2, 2, true>();
}

cudaError_t launch_attn(const Dims& D, const Sess& S, const Pass& P, const DevState& st, const AttnMaps& am, int layer,
                        int tflags, cudaStream_t s) {
  const int max_items = P.full ? 1 : S.max_items;
  cudaError_t e = cudaErrorInvalidValue;
  dim3 cgrid(P.rows_alloc, D.nh);
  const int cthreads = D.hd < 256 ? D.hd : 256;
  if (D.dtype == 1 && (D.hd == 64 || D.hd == 128))
    return D.hd == 64 ? attn_seg_hd<64>(D, S, P, st, am, layer, tflags, s)
                      : attn_seg_hd<128>(D, S, P, st, am, layer, tflags, s);
  if (D.dtype == 1) {
    using T = __nv_bfloat16;
    if (D.hd == 256) e = attn_hd<T, 256>(D, S, P, st, layer, max_items, s);
    else if (D.hd == 32) e = attn_hd<T, 32>(D, S, P, st, layer, max_items, s);
    if (e != cudaSuccess) return e;
    launch_k(k_attn_combine2<T>, dim3(cgrid), dim3(cthreads), (size_t)(0), s, D, S, P, max_items);
  } else {
    using T = float;
    if (D.hd == 64) e = attn_hd<T, 64>(D, S, P, st, layer, max_items, s);
    else if (D.hd == 128) e = attn_hd<T, 128>(D, S, P, st, layer, max_items, s);
    else if (D.hd == 256) e = attn_hd<T, 256>(D, S, P, st, layer, max_items, s);
    else if (D.hd == 32) e = attn_hd<T, 32>(D, S, P, st, layer, max_items, s);
    if (e != cudaSuccess) return e;
    launch_k(k_attn_combine2<T>, dim3(cgrid), dim3(cthreads), (size_t)(0), s, D, S, P, max_items);
  }
  return cudaGetLastError();
}

}  // namespace bb
