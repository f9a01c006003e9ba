// tcgen05 / TMEM / TMA weight-streaming GEMM (bf16 in, fp32 accumulate) and
// the fp32 SIMT GEMM used by fp32 verification mode.
//
// CTA layout (192 threads, 1 CTA per SM):
//   warp 0  lane 0 : TMA producer  (W tile 128x64 + X tile BNx64 per k-block)
//   warp 1  lane 0 : MMA issuer    (4 x tcgen05.mma M128 N=BN K16 per k-block)
//   warps 2-5      : epilogue      (tcgen05.ld TMEM -> regs -> global)
// Two TMEM accumulators (2*BN columns) so the epilogue of one stream-K unit
// overlaps the MMAs of the next.
#include <cudaTypedefs.h>
#include <stdio.h>

#include "bb_common.cuh"
#include "bb_launch.cuh"
#include <cooperative_groups.h>

#include "bb_gemm.cuh"

#ifndef HEAD_T
#define HEAD_T 1  // transposed LM-head epilogue (0: per-row shuffle reductions)
#endif

namespace bb {

struct Unit {
  int tile, kb0, kb1, slot;
};

// Work units of a CTA.  mode 0: stream-K over the flattened (tile, k-block)
// space; mode 0 with np > 0 (compacting sessions): every tile is cut into np
// fixed k-pieces (piece q = plane q) and the pieces are dealt out in
// contiguous runs -- a tile's sums then do not depend on how many row chunks
// the launch computes; mode 1: whole tiles round-robin.
struct UnitIter {
  long long x, end, T;
  int KB, G, c, mode, n_tiles, np;
  __device__ UnitIter(int c_, int G_, int KB_, int n_tiles_, int mode_, int np_ = 0)
      : c(c_), G(G_), KB(KB_), n_tiles(n_tiles_), mode(mode_), np(np_) {
    T = (long long)n_tiles * KB;
    if (mode == 0 && np > 0) {
      const long long TP = (long long)n_tiles * np;
      x = (long long)c * TP / G;
      end = (long long)(c + 1) * TP / G;
    } else if (mode == 0) {
      x = (long long)c * T / G;
      end = (long long)(c + 1) * T / G;
    } else {  // modes 1, 2: whole tiles round-robin
      x = c;
      end = n_tiles;
    }
  }
  __device__ bool next(Unit& u) {
    if (x >= end) return false;
    if (mode != 0) {
      u.tile = (int)x;
      u.kb0 = 0;
      u.kb1 = KB;
      u.slot = 0;
      x += G;
      return true;
    }
    if (np > 0) {
      const int q = (int)(x % np);
      u.tile = (int)(x / np);
      u.kb0 = q * KB / np;
      u.kb1 = (q + 1) * KB / np;
      u.slot = q;
      x += 1;
      return true;
    }
    const int tile = (int)(x / KB);
    const int kb0 = (int)(x % KB);
    const long long rem = end - x;
    const int kb1 = (int)((long long)kb0 + rem < KB ? kb0 + rem : KB);
    u.tile = tile;
    u.kb0 = kb0;
    u.kb1 = kb1;
    u.slot = c - sk_owner((long long)tile * KB, T, G);
    x += kb1 - kb0;
    return true;
  }
};

// One CTA per SM with a deep TMA pipeline (9 x 24 KB stages at BN=64): a
// streaming CTA needs ~100+ KB in flight to pull its share of HBM bandwidth.
// HEAD: the LM-head epilogue's reduction scratch takes a stage's worth of
// shared memory; the stream-K GEMMs use it for one more stage.
template <int BN, bool HEAD>
struct TcCfg {
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int B_BYTES = BN * 128;
  // LM-head epilogue: per-warp (max, argmax, sum) rows + a 32x33 transpose tile per warp
  static constexpr size_t RED = HEAD ? ((size_t)3 * 4 * BN + 4 * 32 * 33) * 4 : 0;
  static constexpr size_t BUDGET = 227 * 1024 - 1024 - 256 - RED;  // dynamic smem for the stages
  static constexpr int STAGES_FIT = (int)(BUDGET / (A_BYTES + B_BYTES));
  static constexpr int STAGES = STAGES_FIT > 10 ? 10 : STAGES_FIT;
  static constexpr uint32_t TCOLS = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * (A_BYTES + B_BYTES) + (2 * STAGES + 4) * 8 + 16 +
                                 RED;
  static_assert(SMEM <= 227 * 1024, "GEMM shared memory");
};

// Tile order.  Stream-K (mode 0): chunk-outer (tile = chunk * n_ntiles +
// ntile; the piece-count tables and consumers assume it).  Whole tiles
// (mode 1, LM head): ntile-outer, so the row chunks of one weight tile run on
// neighbouring CTAs at the same time and the weight tile is read from HBM
// once (chunk-outer would re-stream the 1 GB head once per chunk).
// Mode 2: groups of gc row chunks; inside a group the gc chunks of one weight
// tile are consecutive (ntile-major).  (Walking the fixed pieces of compacting
// sessions ntile-outer the same way measured 1% slower: chunk-outer kept.)
__device__ __forceinline__ int tile_ntile(const GemmTcParams& p, int t, int nch) {
  if (p.mode == 2) {
    const int span = p.n_ntiles * p.gc, g = t / span, gcs = min(p.gc, nch - g * p.gc);
    return (t - g * span) / gcs;
  }
  return p.mode == 1 ? t / nch : t % p.n_ntiles;
}
__device__ __forceinline__ int tile_chunk(const GemmTcParams& p, int t, int nch) {
  if (p.mode == 2) {
    const int span = p.n_ntiles * p.gc, g = t / span, gcs = min(p.gc, nch - g * p.gc);
    return g * p.gc + (t - g * span) % gcs;
  }
  return p.mode == 1 ? t % nch : t / p.n_ntiles;
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ SplitK sk_of(const GemmTcParams& p, int G) {
  SplitK sk;
  sk.KB = p.KB;
  sk.n_chunks = p.n_chunks;
  sk.n_ntiles = p.n_ntiles;
  sk.BN = p.rows_alloc / p.n_chunks;
  sk.G = G;
  sk.T = (long long)p.n_ntiles * p.n_chunks * p.KB;
  sk.ns_tab = nullptr;
  return sk;
}

// LM-head epilogue for 32 rows (per-(row, vocab-tile) max / argmax / sum-exp)
template <int BN>
__device__ __forceinline__ void head_rows(const GemmTcParams& p, float (&v)[32], int n, int q, int lane, int row0, int j0,
                                          float* red) {
  const float hs = p.head_scale, sc = p.spike_cut, sg = p.spike_gain;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int row = row0 + j0 + j;
    float l = -INFINITY;
    if (n < p.n_out && row < p.rows_alloc) {
      l = head_logit(v[j], hs, sc, sg);
      if (n == __ldg(&p.tgt[row])) l += __ldg(&p.boost[row]);
    }
    float m = l;
    int a = n;
    warp_argmax(m, a);
    const float e = (m == -INFINITY) ? 0.0f : expf(l - m);
    const float s = warp_sum(e);
    if (lane == 0) {
      red[(0 * 4 + q) * BN + j0 + j] = m;
      red[(1 * 4 + q) * BN + j0 + j] = __int_as_float(a);
      red[(2 * 4 + q) * BN + j0 + j] = s;
    }
  }
}

// Same statistics, transposed: the warp stages its 32 columns x 32 rows in
// shared memory and lane r reduces row r over the 32 columns sequentially (no
// per-row shuffle trees); ties keep the lowest column as in warp_argmax.  The
// spike and the target boost are applied by the row's lane.
template <int BN>
__device__ __forceinline__ void head_rows_t(const GemmTcParams& p, const float (&v)[32], int n0w, int q, int lane,
                                            int row0, int j0, float* red, float* st) {
#pragma unroll
  for (int j = 0; j < 32; ++j) st[j * 33 + lane] = v[j];
  __syncwarp();
  const int row = row0 + j0 + lane;
  float m = -INFINITY, s = 0.0f;
  int a = n0w;
  if (row < p.rows_alloc) {
    const float hs = p.head_scale, sc = p.spike_cut, sg = p.spike_gain;
    const int tg = __ldg(&p.tgt[row]);
    const float bo = __ldg(&p.boost[row]);
    const int nc = min(32, p.n_out - n0w);
    float l[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      float x = head_logit(st[lane * 33 + c], hs, sc, sg);
      if (n0w + c == tg) x += bo;
      l[c] = c < nc ? x : -INFINITY;
      if (l[c] > m) {
        m = l[c];
        a = n0w + c;
      }
    }
    if (m != -INFINITY) {
#pragma unroll
      for (int c = 0; c < 32; ++c) s += (l[c] == -INFINITY) ? 0.0f : expf(l[c] - m);
    }
  }
  red[(0 * 4 + q) * BN + j0 + lane] = m;
  red[(1 * 4 + q) * BN + j0 + lane] = __int_as_float(a);
  red[(2 * 4 + q) * BN + j0 + lane] = s;
  __syncwarp();
}

#ifndef BB_GEMM_PH
#define BB_GEMM_PH 0  // 1: timeline-session phase marks (GemmTcParams::ph); costs ~1% when built in
#endif
template <int BN, bool HEAD>
__global__ void __launch_bounds__(192)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmB2, const GemmTcParams p) {
  using C = TcCfg<BN, HEAD>;
  namespace cg = cooperative_groups;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* red = reinterpret_cast<float*>(tslot + 4);  // LM-head reduction scratch (HEAD instances)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = p.n_ntiles * p.n_chunks;
  __shared__ int s_pre;  // stages whose weight tile was issued before the dependency wait
  tsite_entry(p.tstat);  // the launch's duration counts from here: the pre-wait weight prefetch included
#if BB_GEMM_PH
  const unsigned long long t_in = p.ph != nullptr ? globaltimer_ns() : 0ull;
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (p.half) tma_prefetch_desc(&tmB2);
  }
  if (warp == 1) tmem_alloc(tslot, C::TCOLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  // PDL: let the next kernel launch, then stream the first weight tiles (which
  // no predecessor writes) while the previous kernel drains; activations (the
  // B tiles) are only touched after the dependency wait.
  pdl_launch();
  if (warp == 0 && lane == 0) {
    // streamed weights are read once (evict first); mode 2 re-reads each weight tile
    // for the gc chunks of its group
    const uint64_t pol_w = p.mode == 2 ? policy_evict_normal() : policy_evict_first();
    int pre = 0;
    UnitIter it(blockIdx.x, gridDim.x, p.KB, n_tiles, p.mode);
    Unit u;
    // (a compacting session's row count is only known after the dependency wait: no prefetch)
    while (p.rows_dyn == nullptr && pre < C::STAGES && it.next(u)) {
      const int ntile = tile_ntile(p, u.tile, p.n_chunks);
      for (int kb = u.kb0; kb < u.kb1 && pre < C::STAGES; ++kb, ++pre) {
        mbar_expect_tx_only(&full[pre], C::A_BYTES);
        tma_load_2d(sA + pre * C::A_BYTES, &tmA, &full[pre], kb * 64, ntile * 128, pol_w);
      }
    }
    s_pre = pre;
  }
  pdl_wait();
  klog_mark(p.klog, p.klog_cap, p.klog_id);
  tsite_begin(p.tstat);
  auto gph = [&](int i) {  // (timeline) ns since this CTA's entry
#if BB_GEMM_PH
    if (p.ph != nullptr) atomicAdd(&p.ph[i], globaltimer_ns() - t_in);
#endif
  };
  if (BB_GEMM_PH && p.ph != nullptr && threadIdx.x == 0) atomicAdd(&p.ph[0], 1ull);
  if (threadIdx.x == 32) gph(1);  // MMA thread: dependency wait returned
  if (threadIdx.x == 0) gph(7);   // producer (issued the weight prefetch first)
  const bool skipped = p.skip != nullptr && *p.skip != 0;
  const int rows_valid = skipped ? 0 : (p.rows_valid != nullptr ? *p.rows_valid : p.rows_alloc);
  // row chunks this launch computes (compacting sessions: the live rows only)
  const int rows_c0 = p.half ? p.half : BN;
  const int nch = p.rows_dyn != nullptr ? min(p.n_chunks, (*p.rows_dyn + rows_c0 - 1) / rows_c0) : p.n_chunks;
  const int n_tiles_eff = p.n_ntiles * nch;
  if (skipped) {
    // drain the prefetched weight tiles before exiting (async copies into our smem)
    __syncthreads();
    if (warp == 0 && lane == 0)
      for (int st = 0; st < s_pre; ++st) {
        mbar_arrive(&full[st]);
        mbar_wait(&full[st], 0);
      }
    __syncthreads();
    if (warp == 1) {
      tc_fence_after();
      tmem_dealloc(tbase, C::TCOLS);
    }
    tsite_end(p.tstat);
    return;
  }

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = p.mode == 2 ? policy_evict_normal() : policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage_i = 0;
      uint32_t phase = 0;
      int issued = 0;  // global k-block counter (matches the prefetch order)
      const int pre = s_pre;
      const int rows_c = p.half ? p.half : BN;  // activation rows per chunk
      // the chunk's activation tile: hi rows (and, bf16x2, the lo rows right after them)
      auto load_b = [&](int st, int kb, int chunk) {
        tma_load_2d(sB + st * C::B_BYTES, &tmB, &full[st], kb * 64, chunk * rows_c, pol_x);
        if (p.half) tma_load_2d(sB + st * C::B_BYTES + p.half * 128, &tmB2, &full[st], kb * 64, chunk * rows_c, pol_x);
      };
      UnitIter it(blockIdx.x, gridDim.x, p.KB, n_tiles_eff, p.mode, p.np);
      Unit u;
      while (it.next(u)) {
        const int ntile = tile_ntile(p, u.tile, nch), chunk = tile_chunk(p, u.tile, nch);
        // (row chunks are never fully padding: rows_alloc = round_up(rows, BN))
        for (int kb = u.kb0; kb < u.kb1; ++kb, ++issued) {
          if (issued < pre) {
            // weight tile already in flight: add the activation tile
            mbar_expect_tx(&full[stage_i], C::B_BYTES);
            load_b(stage_i, kb, chunk);
            if (issued == 0) gph(6);
          } else {
            mbar_wait(&empty[stage_i], phase ^ 1);
            mbar_expect_tx(&full[stage_i], C::A_BYTES + C::B_BYTES);
            tma_load_2d(sA + stage_i * C::A_BYTES, &tmA, &full[stage_i], kb * 64, ntile * 128, pol_w);
            load_b(stage_i, kb, chunk);
          }
          if (++stage_i == C::STAGES) {
            stage_i = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDESC = idesc_bf16_f32(128, BN);
      int stage_i = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      UnitIter it(blockIdx.x, gridDim.x, p.KB, n_tiles_eff, p.mode, p.np);
      Unit u;
      bool first = true;
      while (it.next(u)) {
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t dt = tbase + (uint32_t)(acc * BN);
        for (int kb = u.kb0; kb < u.kb1; ++kb) {
          mbar_wait(&full[stage_i], phase);
          tc_fence_after();
          if (first) {
            gph(2);
            first = false;
          }
          const uint64_t ad = sdesc_sw128(smem_u32(sA + stage_i * C::A_BYTES));
          const uint64_t bd = sdesc_sw128(smem_u32(sB + stage_i * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc_mma_bf16(dt, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), IDESC,
                        (kb > u.kb0 || k > 0) ? 1u : 0u);
          tc_commit(&empty[stage_i]);
          if (++stage_i == C::STAGES) {
            stage_i = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
      gph(3);
    }
  } else {
    const int q = warp & 3;  // TMEM lane quadrant owned by this warp
    const int et = threadIdx.x - 64;
    int acc = 0;
    uint32_t aphase = 0;
    UnitIter it(blockIdx.x, gridDim.x, p.KB, n_tiles_eff, p.mode, p.np);
    Unit u;
    while (it.next(u)) {
      const int ntile = tile_ntile(p, u.tile, nch), chunk = tile_chunk(p, u.tile, nch);
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const int n = ntile * 128 + q * 32 + lane;
      const int rows_c = p.half ? p.half : BN;  // real rows per chunk
      const int row0 = chunk * rows_c;
      const uint32_t taddr = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
      // accumulator columns of real rows [j0, j0+32): bf16x2 folds the lo half in
      auto ld_rows = [&](int j0, float (&v)[32]) {
        tmem_ld32(taddr + j0, v);
        if (p.half) {
          float w[32];
          tmem_ld32(taddr + p.half + j0, w);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += w[j];
        }
      };
      if (p.mode != 1) {
        // stream-K (mode 2: plane 0): raw fp32 partial planes for the post-GEMM kernels
        float* dst = p.part + (long long)u.slot * p.plane + n;
#pragma unroll 1
        for (int j0 = 0; j0 < rows_c; j0 += 32) {
          float v[32];
          ld_rows(j0, v);
          if (n < p.n_out) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int row = row0 + j0 + j;
              if (row < rows_valid) dst[(long long)row * p.ldp] = v[j];
            }
          }
        }
      } else if (HEAD) {
#pragma unroll 1
        for (int j0 = 0; j0 < rows_c; j0 += 32) {
          float v[32];
          ld_rows(j0, v);
          if (p.raw_out != nullptr && n < p.n_out) {  // seams / observers: raw h . w_v per (row, column)
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (row0 + j0 + j < rows_valid) p.raw_out[(long long)(row0 + j0 + j) * p.n_out + n] = v[j];
          }
#if HEAD_T
          head_rows_t<BN>(p, v, ntile * 128 + q * 32, q, lane, row0, j0, red, red + 12 * BN + q * 32 * 33);
#else
          head_rows<BN>(p, v, n, q, lane, row0, j0, red);
#endif
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        epi_bar();
        for (int r = et; r < rows_c; r += 128) {
          const int row = row0 + r;
          float m = red[r];
          int a = __float_as_int(red[4 * BN + r]);
          for (int qq = 1; qq < 4; ++qq) {
            const float mq = red[qq * BN + r];
            if (mq > m) {
              m = mq;
              a = __float_as_int(red[(4 + qq) * BN + r]);
            }
          }
          float s = 0.0f;
          if (m != -INFINITY)
            for (int qq = 0; qq < 4; ++qq) {
              const float mq = red[qq * BN + r];
              if (mq != -INFINITY) s += red[(8 + qq) * BN + r] * expf(mq - m);
            }
          if (row < rows_valid) p.head_part[(long long)row * p.n_ntiles + ntile] = make_float4(m, __int_as_float(a), s, 0.0f);
        }
        epi_bar();
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
        continue;
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (et == 0 && acc == 0 && aphase == 0) gph(4);  // first tile stored
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, C::TCOLS);
  }
  if (threadIdx.x == 0) gph(5);
  tsite_end(p.tstat);
}

// ------------------------------------------------------------------ host
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static bool get_encode() {
  if (g_encode) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || fn == nullptr)
    return false;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

static bool make_tmap(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_outer) {
  if (!get_encode()) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool tma_map_bf16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_outer) {
  return make_tmap(m, base, inner, outer, box_outer);
}

bool tc_gemm_setup(TcGemm& g, const void* W, int n_out, int K, const void* X, int rows_alloc, int BN, int mode,
                   int max_grid, const void* X_lo) {
  const int mma_n = X_lo != nullptr ? 2 * BN : BN;  // bf16x2: hi + lo rows of a chunk in one MMA
  if (mma_n != 64 && mma_n != 128 && mma_n != 160 && mma_n != 192 && mma_n != 256) return false;
  if (BN % 32 != 0) return false;  // the epilogue reads 32 accumulator columns (rows) at a time
  if (K % 8 != 0) return false;  // 16-byte row stride for TMA
  memset(&g, 0, sizeof(g));
  g.BN = mma_n;
  g.W = W;
  if (!make_tmap(&g.tmA, W, (uint64_t)K, (uint64_t)n_out, 128)) return false;
  if (!make_tmap(&g.tmB, X, (uint64_t)K, (uint64_t)rows_alloc, (uint32_t)BN)) return false;
  if (X_lo != nullptr && !make_tmap(&g.tmB2, X_lo, (uint64_t)K, (uint64_t)rows_alloc, (uint32_t)BN)) return false;
  if (X_lo == nullptr) g.tmB2 = g.tmB;  // never read
  GemmTcParams& p = g.p;
  p.half = X_lo != nullptr ? BN : 0;
  p.n_out = n_out;
  p.K = K;
  p.n_ntiles = (n_out + 127) / 128;
  p.n_chunks = (rows_alloc + BN - 1) / BN;
  p.KB = (K + 63) / 64;
  p.mode = mode;
  p.rows_alloc = rows_alloc;
  p.ldp = n_out;
  p.plane = (long long)rows_alloc * n_out;
  const long long n_tiles = (long long)p.n_ntiles * p.n_chunks;
  const long long T = n_tiles * p.KB;
  const int resident = max_grid > 0 ? max_grid : 148;  // one CTA per SM (TcCfg smem budget)
  if (mode == 1) p.epi.kind = 1;  // LM-head epilogue
  if (mode == 0) {
    const int gmax = resident;
    g.grid = (int)(T < gmax ? T : gmax);
  } else {
    const int gmax = max_grid > 0 ? max_grid : resident;
    const long long rounds = (n_tiles + gmax - 1) / gmax;
    g.grid = (int)((n_tiles + rounds - 1) / rounds);
  }
  g.sk.T = mode == 0 ? T : 0;
  g.sk.KB = p.KB;
  g.sk.G = g.grid;
  g.sk.n_chunks = p.n_chunks;
  g.sk.n_ntiles = p.n_ntiles;
  g.sk.BN = BN;
  g.sk.ns_tab = nullptr;
  g.max_slots = 1;
  if (mode == 0)
    for (long long t = 0; t < n_tiles; ++t) {
      const int ns = sk_owner(t * p.KB + p.KB - 1, T, g.grid) - sk_owner(t * p.KB, T, g.grid) + 1;
      if (ns > g.max_slots) g.max_slots = ns;
    }
  return true;
}

template <int BN, bool HEAD>
static cudaError_t launch_bn(const TcGemm& g, cudaStream_t s) {
  using C = TcCfg<BN, HEAD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_tc<BN, HEAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  launch_k(k_gemm_tc<BN, HEAD>, dim3(g.grid), dim3(192), (size_t)C::SMEM, s, g.tmA, g.tmB, g.tmB2, g.p);
  return cudaGetLastError();
}

template <bool HEAD>
static cudaError_t launch_mode(const TcGemm& g, cudaStream_t s) {
  switch (g.BN) {
    case 64: return launch_bn<64, HEAD>(g, s);
    case 128: return launch_bn<128, HEAD>(g, s);
    case 160: return launch_bn<160, HEAD>(g, s);
    case 192: return launch_bn<192, HEAD>(g, s);
    case 256: return launch_bn<256, HEAD>(g, s);
  }
  return cudaErrorInvalidValue;
}

void tc_gemm_round_robin(TcGemm& g, int min_rounds, int act_row_bytes) {
  GemmTcParams& p = g.p;
  if (p.mode != 0 || (long long)p.n_ntiles * p.n_chunks < (long long)min_rounds * g.grid) return;
  p.mode = 2;
  // a group's activations (gc chunks x rows x K, both planes) ~ 32 MB of L2
  const long long chunk_bytes = (long long)(p.half ? p.half : g.BN) * act_row_bytes;
  long long gc = (32ll << 20) / (chunk_bytes > 0 ? chunk_bytes : 1);
  p.gc = (int)(gc < 4 ? 4 : (gc > 16 ? 16 : gc));
  g.sk.np = 1;  // one piece per tile: the consumers read plane 0 only
  g.max_slots = 1;
}

cudaError_t tc_gemm_launch(const TcGemm& g, cudaStream_t s) {
  return g.p.mode == 1 ? launch_mode<true>(g, s) : launch_mode<false>(g, s);
}

// ------------------------------------------------------------------ SIMT fp32
// out[row][n] = sum_k X[row][k] * W[n][k]; 64x64 tile, 256 threads, 4x4 per thread.
__global__ void __launch_bounds__(256) k_gemm_simt(SimtGemm g) {
  pdl_enter();
  if (g.skip != nullptr && *g.skip != 0) return;
  const int rows = g.rows_valid != nullptr ? *g.rows_valid : g.rows_alloc;
  const int r0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  if (r0 >= rows) return;
  __shared__ float sX[16][64 + 4];
  __shared__ float sW[16][64 + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      const int rr = i / 16, kk = i % 16;
      const int row = r0 + rr, n = n0 + rr, k = k0 + kk;
      sX[kk][rr] = (row < rows && k < g.K) ? g.X[(long long)row * g.K + k] : 0.0f;
      sW[kk][rr] = (n < g.n_out && k < g.K) ? g.W[(long long)n * g.K + k] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = sX[kk][ty * 4 + i];
        b[i] = sW[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = r0 + ty * 4 + i;
    if (row >= rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < g.n_out) g.out[(long long)row * g.ldo + n] = acc[i][j];
    }
  }
}

cudaError_t simt_gemm_launch(const SimtGemm& g, cudaStream_t s) {
  dim3 grid((g.n_out + 63) / 64, (g.rows_alloc + 63) / 64);
  launch_k(k_gemm_simt, dim3(grid), dim3(256), (size_t)(0), s, g);
  return cudaGetLastError();
}

}  // namespace bb
