// Device-side control of the BlockBatch step (scheduler.py:225-394, Alg. 1/2).
//
// One CTA per request runs the sequential decision logic exactly as the
// reference orders it (index order, first-max tie rules, strict/non-strict
// comparisons of SURVEY Appendix A); CTA-wide scans (masks, compatibility,
// EOS) use all threads.  Branch rows live in shared memory during a kernel.
//
// Kernels
//   k_prefill_init   fresh rows, windows, page tables (branch 0 owns the
//                    prefill pages, all others alias them), full-pass slots
//   k_prefill_post   charge init, per-branch Eq. 1 commit, advance
//   k_block_pack     hard cap, active set, copy-on-write of window pages,
//                    block-pass slots + target boost, attention items, charge
//   k_step_commit    Eq. 1 commit per active branch, EOS cycle, early return
//   k_merge_prep     P_d(i, v) for every merge candidate (parallel, from the
//                    stored head input h, m, s, boost)
//   k_merge_sync     Alg. 2 merge + leader sync (page aliasing), refresh due,
//                    final winner
//   k_refresh_pack / k_refresh_end   periodic full refresh (one branch/pass)
//   k_copy_pages     executes page copy-on-write and prob-map copy jobs
#include "bb200.h"
#include "bb_common.cuh"
#include "bb_launch.cuh"
#include "bb_layers.cuh"

namespace bb {

// ------------------------------------------------------------------ CTA helpers
__device__ __forceinline__ int cta_sum(int v, int* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  int t = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  __syncthreads();
  return t;
}
__device__ __forceinline__ int cta_min(int v, int* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  int t = 0x7fffffff;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = min(t, red[w]);
  __syncthreads();
  return t;
}

// CTA-wide (max value, lowest index); invalid lanes pass v = -inf, idx = INT_MAX.
__device__ __forceinline__ int cta_argmax_first(float v, int idx, float* redf, int* redi) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    redf[threadIdx.x >> 5] = v;
    redi[threadIdx.x >> 5] = idx;
  }
  __syncthreads();
  float bv = redf[0];
  int bi = redi[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
    if (redf[w] > bv || (redf[w] == bv && redi[w] < bi)) {
      bv = redf[w];
      bi = redi[w];
    }
  __syncthreads();
  return bi;
}

struct RC {  // request context
  const Dims* D;
  const Sess* S;
  DevState st;
  int r;
  int* rows;   // smem [B][L]
  int* br;     // smem [B][B_WORDS]
  int* ctrl;   // global
  int* red;    // smem [32]
  int mask_id, eos_id;

  __device__ int* row(int k) { return rows + k * S->L; }
  __device__ int& B_(int k, int f) { return br[k * B_WORDS + f]; }

  __device__ bool has_mask(int k, int lo, int hi) {
    int f = 0;
    const int* rw = row(k);
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) f |= (rw[i] == mask_id);
    return __syncthreads_or(f) != 0;
  }
  __device__ int first_mask(int k, int lo, int hi) {  // hi if none
    int f = 0x7fffffff;
    const int* rw = row(k);
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x)
      if (rw[i] == mask_id) {
        f = i;
        break;
      }
    const int m = cta_min(f, red);
    return m == 0x7fffffff ? hi : m;
  }
  __device__ int count_decoded(int k) {  // BranchState.refresh_decoded (decoding.py:91-93)
    int c = 0;
    const int* rw = row(k);
    for (int i = S->P + threadIdx.x; i < S->L; i += blockDim.x) c += (rw[i] != mask_id);
    return cta_sum(c, red);
  }
  __device__ int earliest_eos(int k) {  // decoding.py:157-160, -1 if none
    int f = 0x7fffffff;
    const int* rw = row(k);
    for (int i = S->P + threadIdx.x; i < S->L; i += blockDim.x)
      if (rw[i] == eos_id) {
        f = i;
        break;
      }
    const int m = cta_min(f, red);
    return m == 0x7fffffff ? -1 : m;
  }
  // 0 none, 1 pending, 2 ready (decoding.py:163-168)
  __device__ int check_eos(int k, int* eos_out) {
    const int e = earliest_eos(k);
    if (eos_out) *eos_out = e;
    if (e < 0) return 0;
    return has_mask(k, S->P, e) ? 1 : 2;
  }
  __device__ bool window_complete(int k) {  // decoding.py:137-140
    const int s = B_(k, B_START), e = B_(k, B_END);
    if (s >= e) return true;
    return !has_mask(k, s, e);
  }
  __device__ void advance_while_complete(int k) {  // decoding.py:143-154 in a while loop
    while (true) {
      const bool done = B_(k, B_DONE) != 0;
      if (done || !window_complete(k)) break;
      __syncthreads();
      if (threadIdx.x == 0) {
        const int st0 = B_(k, B_END);
        if (st0 >= S->L) {
          B_(k, B_START) = S->L;
          B_(k, B_END) = S->L;
          B_(k, B_DONE) = 1;
        } else {
          B_(k, B_START) = st0;
          B_(k, B_END) = min(st0 + B_(k, B_SIZE), S->L);
        }
      }
      __syncthreads();
    }
  }
  __device__ void realign_for_eos(int k) {  // decoding.py:171-180
    const int e = earliest_eos(k);
    if (e < 0) return;
    const int f = first_mask(k, 0, e);
    if (f >= e) return;
    __syncthreads();
    if (threadIdx.x == 0) {
      B_(k, B_START) = f;
      B_(k, B_END) = min(f + B_(k, B_SIZE), e);
    }
    __syncthreads();
  }
  __device__ void realign_to_first_mask(int k) {  // decoding.py:183-191
    const int f = first_mask(k, 0, S->L);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (f >= S->L) {
        B_(k, B_START) = S->L;
        B_(k, B_END) = S->L;
        B_(k, B_DONE) = 1;
      } else {
        B_(k, B_START) = f;
        B_(k, B_END) = min(f + B_(k, B_SIZE), S->L);
      }
    }
    __syncthreads();
  }
  __device__ bool compatible(int a, int b) {  // scheduler.py:139-141
    int bad = 0;
    const int *ra = row(a), *rb = row(b);
    for (int i = threadIdx.x; i < S->L; i += blockDim.x) {
      const int x = ra[i], y = rb[i];
      bad |= (x != mask_id && y != mask_id && x != y);
    }
    return __syncthreads_or(bad) == 0;
  }
  __device__ int leader() {  // scheduler.py:212-213: first max of (decoded, -block_size)
    int best = 0;
    for (int k = 1; k < S->B; ++k) {
      const int dk = B_(k, B_DEC), db = B_(best, B_DEC);
      if (dk > db || (dk == db && -B_(k, B_SIZE) > -B_(best, B_SIZE))) best = k;
    }
    return best;
  }
  // thread 0 only
  __device__ void emit(int kind, int branch, int a0 = 0, int a1 = 0, int a2 = 0, int a3 = 0, float prob = 0.0f) {
    if (!S->trace) return;
    const int n = ctrl[C_NEV];
    if (n >= S->ev_cap) {
      ctrl[C_EV_OVERFLOW] = 1;
      return;
    }
    int* e = st.events + ((long long)r * S->ev_cap + n) * EVW;
    e[E_KIND] = kind;
    e[E_BRANCH] = branch;
    e[E_NFE0] = ctrl[C_NFE0];
    e[E_NFE1] = ctrl[C_NFE1];
    e[E_NFE2] = ctrl[C_NFE2];
    e[E_A0] = a0;
    e[E_A1] = a1;
    e[E_A2] = a2;
    e[E_A3] = a3;
    e[E_PROB] = __float_as_int(prob);
    for (int k = 0; k < MAXB; ++k) e[E_DEC + k] = k < S->B ? B_(k, B_DEC) : 0;
    ctrl[C_NEV] = n + 1;
  }
  // ---- page manager (thread 0 only) ----
  __device__ int* pt(int k) { return st.pt + ((long long)r * S->B + k) * S->n_lp; }
  __device__ int* refc() { return st.refc + (long long)r * S->pool; }
  __device__ int pg_alloc() {
    int& top = st.free_top[r];
    if (top <= 0) {
      ctrl[C_STATUS] = BB_ERR_STATE;
      return 0;
    }
    --top;
    const int p = st.freel[(long long)r * S->pool + top];
    refc()[p] = 1;
    return p;
  }
  __device__ void pg_decref(int p) {
    if (--refc()[p] == 0) st.freel[(long long)r * S->pool + st.free_top[r]++] = p;
  }
  // make (k, lp) private before a write; copy the old contents iff `copy`
  __device__ void write_intent(int k, int lp, bool copy) {
    int* t = pt(k);
    const int p = t[lp];
    if (refc()[p] <= 1) return;
    const int np = pg_alloc();
    if (copy) {
      const int n = ctrl[C_NCOPY];
      if (n < S->max_copies) {
        st.copies[((long long)r * S->max_copies + n) * 2] = p;
        st.copies[((long long)r * S->max_copies + n) * 2 + 1] = np;
        ctrl[C_NCOPY] = n + 1;
      } else {
        ctrl[C_STATUS] = BB_ERR_STATE;
      }
      ctrl[C_COW_PAGES] += 1;
    }
    refc()[p] -= 1;
    t[lp] = np;
  }
};

__device__ void load_request(RC& c) {
  const int n = c.S->B * c.S->L;
  const int* g = c.st.tokens + (long long)c.r * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) c.rows[i] = g[i];
  const int nb = c.S->B * B_WORDS;
  const int* gb = c.st.br + (long long)c.r * nb;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) c.br[i] = gb[i];
  __syncthreads();
}
__device__ void store_request(RC& c) {
  __syncthreads();
  const int n = c.S->B * c.S->L;
  int* g = c.st.tokens + (long long)c.r * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) g[i] = c.rows[i];
  const int nb = c.S->B * B_WORDS;
  int* gb = c.st.br + (long long)c.r * nb;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) gb[i] = c.br[i];
  __syncthreads();
}

#define RC_SETUP()                                                   \
  extern __shared__ int smem_i[];                                    \
  __shared__ int red[32];                                            \
  __shared__ int sbr[MAXB * B_WORDS];                                \
  RC c;                                                              \
  c.D = &D;                                                          \
  c.S = &S;                                                          \
  c.st = st;                                                         \
  c.r = blockIdx.x;                                                  \
  c.rows = smem_i;                                                   \
  c.br = sbr;                                                        \
  c.ctrl = st.ctrl + (long long)blockIdx.x * C_WORDS;                \
  c.red = red;                                                       \
  c.mask_id = D.V + 1;                                               \
  c.eos_id = D.V;

// element offset (within one layer) of the K/V row of (request r, branch k, pos)
__device__ __forceinline__ long long kv_row_off(const Dims& D, const Sess& S, const DevState& st, int r, int k, int pos) {
  const int lp = lp_of(S, pos);
  const long long gpage = (long long)r * S.pool + st.pt[((long long)r * S.B + k) * S.n_lp + lp];
  return (gpage * D.nkv * S.ps + (pos - lp_start(S, lp))) * D.hd;
}

// boost / target of a head slot at `pos` of row `rw` (model.py:258-275, 306-317)
__device__ void slot_boost(const Dims& D, const Sess& S, const int* rw, const int* target, int pos, float* boost,
                           int* tgt) {
  const int mask_id = D.V + 1;
  if (pos < S.P || target == nullptr) {  // prompt position (seams) / no target: not predictable (model.py:310-317)
    *boost = 0.0f;
    *tgt = -1;
    return;
  }
  const int t = target[pos - S.P];
  const int lo = max(pos - D.radius, 0), hi = min(pos + D.radius + 1, S.L);
  int nc = 0, nm = 0;
  for (int j = lo; j < hi; ++j) {
    if (j == pos) continue;
    const int x = rw[j];
    if (x == mask_id) continue;
    ++nc;
    const int ft = j < S.P ? x : target[j - S.P];
    nm += (x == ft);
  }
  const float ag = nc > 0 ? (float)nm / (float)nc : 0.0f;
  *boost = D.gamma != 0.0f ? D.gamma * ag : 0.0f;
  *tgt = (t <= D.V) ? t : -1;
}

// ------------------------------------------------------------------ prefill
__global__ void k_prefill_init(Dims D, Sess S, DevState st, Pass full, Pass blk, Head H) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 10);
  RC_SETUP();
  const int r = c.r;
  const int* prompt = st.prompt + (long long)r * S.P;
  const int* init_gen = st.init_gen + (long long)r * S.G;  // presets (decoding.py:194-200), -1 = mask
  for (int k = 0; k < S.B; ++k)
    for (int i = threadIdx.x; i < S.L; i += blockDim.x)
      c.rows[k * S.L + i] = i < S.P ? prompt[i] : (init_gen[i - S.P] >= 0 ? init_gen[i - S.P] : c.mask_id);
  if (threadIdx.x < C_WORDS) c.ctrl[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    int n_preset = 0;  // refresh_decoded counts them before the first forward (decoding.py:212-218)
    for (int i = 0; i < S.G; ++i) n_preset += init_gen[i] >= 0;
    for (int k = 0; k < S.B; ++k) {
      c.B_(k, B_START) = S.P;
      c.B_(k, B_END) = min(S.P + S.bs[k], S.L);
      c.B_(k, B_DONE) = 0;
      c.B_(k, B_DEC) = n_preset;
      c.B_(k, B_MERGED) = 0;
      c.B_(k, B_SIZE) = S.bs[k];
      c.B_(k, 6) = 0;
      c.B_(k, 7) = 0;
    }
  }
  for (int i = threadIdx.x; i < S.B * S.L; i += blockDim.x) st.covered[(long long)r * S.B * S.L + i] = 0;
  // page pool: free stack pops 0,1,2...; a diagnostics session keeps the last
  // n_lp pages out of it (scratch for bb_fresh_kv)
  const int n_free = S.pool - (S.diag ? S.n_lp : 0);
  for (int i = threadIdx.x; i < S.pool; i += blockDim.x) {
    st.freel[(long long)r * S.pool + i] = n_free - 1 - i;
    st.refc[(long long)r * S.pool + i] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    st.free_top[r] = n_free;
    int* t0 = c.pt(0);
    for (int lp = 0; lp < S.n_lp; ++lp) t0[lp] = c.pg_alloc();
    for (int k = 1; k < S.B; ++k) {
      int* tk = c.pt(k);
      for (int lp = 0; lp < S.n_lp; ++lp) {
        tk[lp] = t0[lp];
        c.refc()[t0[lp]] += 1;
      }
    }
    c.ctrl[C_SHARED_PAGES] = S.n_lp;
    for (int k = 0; k < MAXB; ++k) {
      full.rng_off[r * MAXB + k] = r * S.L;
      full.rng_cnt[r * MAXB + k] = k == 0 ? S.L : 0;
    }
    full.n_items[r] = 1;
    int* it = full.items + (long long)r * ITW;
    it[0] = 1;
    it[1] = 0;
    it[2] = S.n_lp;
    it[3] = 0;
    *full.skip = 0;
    *H.skip = 0;
  }
  __syncthreads();
  // full-pass rows: the shared base row (branch 0)
  for (int p = threadIdx.x; p < S.L; p += blockDim.x) {
    const int row = r * S.L + p;
    full.slot_pos[row] = p;
    full.slot_req[row] = r;
    full.slot_br[row] = 0;
    full.slot_tok[row] = c.rows[p];
    full.slot_kvoff[row] = kv_row_off(D, S, st, r, 0, p);
  }
  // head slots: each branch's initial window over the base row (every request
  // is live at prefill: the static slot layout, also restored for compaction)
  if (threadIdx.x == 0) {
    blk.req_base[r] = r * S.NRq;
    if (r == 0) *blk.rows_live = S.NR;
  }
  const int* target = st.target + (long long)r * S.G;
  for (int i = threadIdx.x; i < S.NRq; i += blockDim.x) {
    const int slot = r * S.NRq + i;
    int k = -1;
    for (int kk = 0; kk < S.B; ++kk)
      if (i >= S.off[kk] && i < S.off[kk] + S.bs[kk]) k = kk;
    int pos = -1;
    if (k >= 0) {
      const int j = i - S.off[k];
      if (S.P + j < c.B_(k, B_END)) pos = S.P + j;
    }
    blk.slot_req[slot] = r;
    blk.slot_br[slot] = k < 0 ? 0 : k;
    blk.slot_pos[slot] = pos;
    H.masked[slot] = (pos >= 0 && c.rows[pos] == c.mask_id) ? 1 : 0;  // preset positions are not queried
    if (pos >= 0) slot_boost(D, S, c.rows, target, pos, &H.boost[slot], &H.tgt[slot]);
    else {
      H.boost[slot] = 0.0f;
      H.tgt[slot] = -1;
    }
  }
  store_request(c);
}

// Eq. 1 (decoding.py:108-129) over n candidate rows in position order:
// i* = first max of conf (lowest position), commit iff conf >= tau or i == i*;
// the committed token is the (lowest-id) argmax.  Thread 0.  Returns #commits;
// writes (pos, tok) pairs to `out` if non-null.
__device__ int eq1_commit(const float* conf, const int* arg, const int* pos, const int* valid, int n, float tau,
                          int* row, int* out) {
  int star = -1;
  float best = 0.0f;
  for (int j = 0; j < n; ++j) {
    if (!valid[j]) continue;
    if (star < 0 || conf[j] > best) {
      star = j;
      best = conf[j];
    }
  }
  if (star < 0) return 0;
  int cnt = 0;
  for (int j = 0; j < n; ++j) {
    if (!valid[j]) continue;
    if (conf[j] >= tau || j == star) {
      row[pos[j]] = arg[j];
      if (out) {
        out[2 * cnt] = pos[j];
        out[2 * cnt + 1] = arg[j];
      }
      ++cnt;
    }
  }
  return cnt;
}

// Eq. 1 for branch k over its head slots, CTA-parallel: i* = first max conf
// (lowest position), commit iff conf >= tau or i == i*.  All threads call;
// returns #commits.
__device__ int apply_commits(RC& c, const Pass& blk, const Head& H, int k, float tau) {
  __shared__ float redf[32];
  __shared__ int redi[32];
  const int slot0 = blk_base(*c.S, blk, c.r) + c.S->off[k];
  const int n = c.S->bs[k];
  int star = 0x7fffffff;
  for (int base = 0; base < n; base += blockDim.x) {
    const int j = base + threadIdx.x;
    const bool valid = j < n && H.masked[slot0 + j];
    const float cf = valid ? H.res_conf[slot0 + j] : -INFINITY;
    const int cand = cta_argmax_first(cf, valid ? j : 0x7fffffff, redf, redi);
    if (cand != 0x7fffffff) {
      // combine with previous bases (earlier j wins ties)
      if (star == 0x7fffffff || H.res_conf[slot0 + cand] > H.res_conf[slot0 + star]) star = cand;
    }
  }
  if (star == 0x7fffffff) return 0;
  int cnt = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int j = base + threadIdx.x;
    bool commit = false;
    if (j < n && H.masked[slot0 + j]) {
      const int slot = slot0 + j;
      commit = H.res_conf[slot] >= tau || j == star;
      if (commit) c.row(k)[blk.slot_pos[slot]] = H.res_arg[slot];
    }
    cnt += __syncthreads_count(commit);
  }
  return cnt;
}

__global__ void k_prefill_post(Dims D, Sess S, DevState st, Pass blk, Head H) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 11);
  RC_SETUP();
  load_request(c);
  if (c.ctrl[C_STATUS] != 0) return;
  __shared__ int s_n;
  if (threadIdx.x == 0) {
    c.ctrl[C_NFE0] += 1;
    c.emit(EV_INIT, -1);
  }
  for (int k = 0; k < S.B; ++k) {
    if (threadIdx.x == 0) s_n = -1;
    __syncthreads();
    const bool any = c.has_mask(k, c.B_(k, B_START), c.B_(k, B_END));
    if (any) {
      const int nc = apply_commits(c, blk, H, k, S.tau_conf);
      if (threadIdx.x == 0) s_n = nc;
    }
    __syncthreads();
    if (any) {
      const int dec = c.count_decoded(k);
      if (threadIdx.x == 0) {
        c.B_(k, B_DEC) = dec;
        c.ctrl[C_COMMITS] += s_n;
        c.emit(EV_DECODE, k, s_n);
      }
      __syncthreads();
    }
  }
  for (int k = 0; k < S.B; ++k) c.advance_while_complete(k);
  store_request(c);
}

// ------------------------------------------------------------------ block step
// Block pass of the branches in `active` (all threads call; thread 0 does
// the page work): copy-on-write of the window pages (model.py:289
// copy-then-write), the SIMT attention items (active branches grouped by
// physical page), the per-branch row ranges and the head slots (window
// positions; masked ones report to the LM head).
__device__ void pack_block_pass(RC& c, int active, const Pass& blk, const Head& H, const int* target) {
  const Dims& D = *c.D;
  const Sess& S = *c.S;
  const int r = c.r;
  const int base = blk_base(S, blk, r);  // -1: a finished request of a compacting session (no slots)
  if (threadIdx.x == 0) {
    c.ctrl[C_NCOPY] = 0;
    if (active) {
      for (int k = 0; k < S.B; ++k) {
        if (!((active >> k) & 1) || c.B_(k, B_START) >= c.B_(k, B_END)) continue;
        const int lp0 = lp_of(S, c.B_(k, B_START)), lp1 = lp_of(S, c.B_(k, B_END) - 1);
        for (int lp = lp0; lp <= lp1; ++lp) c.write_intent(k, lp, true);
      }
      // SIMT attention items: the logical pages split into fixed runs of
      // ch_block pages; active branches whose run maps to the same physical
      // pages share one item.  A row's key partition (and so its partials'
      // combine order) is the same whatever pages its branch shares, so a
      // branch's block forward is bitwise the same batched or alone
      // (scheduler.py:116-131, test_scheduler.py:72-91).
      int n_items = 0, shared_pages = 0;
      const int n_runs = uses_items(D) ? (S.n_lp + S.ch_block - 1) / S.ch_block : 0;
      for (int run = 0; run < n_runs; ++run) {
        const int lp0 = run * S.ch_block, lp1 = min(lp0 + S.ch_block, S.n_lp);
        int done_mask = 0;
        for (int k = 0; k < S.B; ++k) {
          if (!((active >> k) & 1) || ((done_mask >> k) & 1)) continue;
          int m = 0;
          for (int k2 = k; k2 < S.B; ++k2) {
            if (!((active >> k2) & 1)) continue;
            bool same = true;
            for (int lp = lp0; lp < lp1 && same; ++lp) same = c.pt(k2)[lp] == c.pt(k)[lp];
            if (same) m |= 1 << k2;
          }
          done_mask |= m;
          if (__popc(m) > 1) shared_pages += lp1 - lp0;
          if (n_items < S.max_items) {
            int* ni = blk.items + ((long long)r * S.max_items + n_items) * ITW;
            ni[0] = m;
            ni[1] = lp0;
            ni[2] = lp1;
            ni[3] = k;
            ++n_items;
          } else {
            c.ctrl[C_STATUS] = BB_ERR_STATE;
          }
        }
      }
      blk.n_items[r] = n_items;
      c.ctrl[C_SHARED_PAGES] = shared_pages;
      *blk.skip = 0;
      *H.skip = 0;
    } else {
      blk.n_items[r] = 0;
    }
    int rows = 0;
    for (int k = 0; k < MAXB; ++k) {
      const bool a = k < S.B && ((active >> k) & 1);
      blk.rng_off[r * MAXB + k] = base + (k < S.B ? S.off[k] : 0);
      blk.rng_cnt[r * MAXB + k] = a ? c.B_(k, B_END) - c.B_(k, B_START) : 0;
      rows += blk.rng_cnt[r * MAXB + k];
    }
    c.ctrl[C_BLOCK_ROWS] = rows;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < S.NRq && base >= 0; i += blockDim.x) {
    const int slot = base + i;
    int k = -1;
    for (int kk = 0; kk < S.B; ++kk)
      if (i >= S.off[kk] && i < S.off[kk] + S.bs[kk]) k = kk;
    int pos = -1;
    if (k >= 0 && ((active >> k) & 1)) {
      const int j = i - S.off[k];
      if (c.B_(k, B_START) + j < c.B_(k, B_END)) pos = c.B_(k, B_START) + j;
    }
    blk.slot_req[slot] = r;
    blk.slot_br[slot] = k < 0 ? 0 : k;
    blk.slot_pos[slot] = pos;
    const int tok = pos >= 0 ? c.rows[k * S.L + pos] : 0;
    blk.slot_tok[slot] = tok;
    blk.slot_kvoff[slot] = pos >= 0 ? kv_row_off(D, S, c.st, r, k, pos) : 0;
    const int msk = pos >= 0 && tok == c.mask_id;
    H.masked[slot] = msk;
    if (msk) slot_boost(D, S, c.rows + k * S.L, target, pos, &H.boost[slot], &H.tgt[slot]);
    else {
      H.boost[slot] = 0.0f;
      H.tgt[slot] = -1;
    }
  }
}

// Compacting sessions: the block pass's slots go to the live requests only,
// in request order (request r's NRq slots start at rank(r) * NRq), and the
// GEMMs / head size their work by rows_live -- finished requests of a batch
// cost no rows.  Slots past rows_live are cleared (padding).  One CTA.
__global__ void k_block_bases(Dims D, Sess S, DevState st, Pass blk, Head H) {
  pdl_enter();
  __shared__ int s_live;
  if (threadIdx.x == 0) {
    int n = 0;
    for (int r = 0; r < S.R; ++r) {
      const bool live = st.ctrl[(long long)r * C_WORDS + C_STATUS] == 0;
      blk.req_base[r] = live ? n * S.NRq : -1;
      n += live ? 1 : 0;
    }
    s_live = n * S.NRq;
    *blk.rows_live = s_live;
  }
  __syncthreads();
  for (int slot = s_live + (int)threadIdx.x; slot < S.NR; slot += blockDim.x) {
    blk.slot_pos[slot] = -1;
    H.masked[slot] = 0;
  }
}

__global__ void k_block_pack(Dims D, Sess S, DevState st, Pass blk, Head H) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 12);
  RC_SETUP();
  const int r = c.r;
  __shared__ int s_active, s_live;
  load_request(c);
  if (threadIdx.x == 0) {
    s_live = c.ctrl[C_STATUS] == 0;
    if (s_live) {
      c.ctrl[C_ITER] += 1;
      const int total = c.ctrl[C_NFE0] + c.ctrl[C_NFE1] + c.ctrl[C_NFE2];
      if (total > S.hard_cap || c.ctrl[C_ITER] > 10 * S.hard_cap) {
        c.ctrl[C_STATUS] = BB_ERR_RUNAWAY;
        s_live = 0;
      } else if (c.ctrl[C_REFRESH_DUE]) {
        c.ctrl[C_STATUS] = BB_ERR_STATE;  // host skipped a due refresh
        s_live = 0;
      }
    }
    s_active = 0;
  }
  __syncthreads();
  if (s_live) {
    for (int k = 0; k < S.B; ++k) {
      if (c.B_(k, B_DONE)) continue;
      if (c.has_mask(k, c.B_(k, B_START), c.B_(k, B_END)) && threadIdx.x == 0) s_active |= 1 << k;
    }
  }
  __syncthreads();
  const int active = s_active;
  if (threadIdx.x == 0) {
    c.ctrl[C_ACTIVE_MASK] = active;
    if (active) {
      c.ctrl[C_NFE1] += 1;
      c.ctrl[C_SINCE_REFRESH] += 1;
      c.ctrl[C_LAST_ACTIVE] = active;
      c.emit(EV_BLOCK, -1, active);
    }
  }
  pack_block_pass(c, active, blk, H, st.target + (long long)r * S.G);
  store_request(c);
}

// ------------------------------------------------------------------ step-operator seams
// Seam sessions (model.py:322-343 full_forward / block_forward, scheduler.py:
// 80-89 init_full_forward, 116-131 batched_block_forward): every branch owns
// private pages [k*n_lp, (k+1)*n_lp) (the caller loads its cache into them);
// no NFE accounting, no events.
__global__ void k_seam_init(Dims D, Sess S, DevState st) {
  pdl_enter();
  const int r = blockIdx.x;
  if (threadIdx.x < C_WORDS) st.ctrl[(long long)r * C_WORDS + threadIdx.x] = 0;
  for (int i = threadIdx.x; i < S.pool; i += blockDim.x) {
    const bool own = i < S.B * S.n_lp;
    st.refc[(long long)r * S.pool + i] = own ? 1 : 0;
    // free stack: the pages no branch owns (diagnostics scratch excluded)
    const int n_free = S.pool - S.B * S.n_lp - (S.diag ? S.n_lp : 0);
    if (i < n_free) st.freel[(long long)r * S.pool + i] = S.B * S.n_lp + i;
  }
  for (int i = threadIdx.x; i < S.B * S.n_lp; i += blockDim.x) st.pt[(long long)r * S.B * S.n_lp + i] = i;
  if (threadIdx.x == 0) st.free_top[r] = S.pool - S.B * S.n_lp - (S.diag ? S.n_lp : 0);
}

// block_forward of the branches in `mask` over their windows [start, end)
// (whether or not the window holds a mask: the reference recomputes the
// window's K/V regardless, model.py:331-343)
__global__ void k_seam_block_pack(Dims D, Sess S, DevState st, Pass blk, Head H, int mask, int use_target) {
  pdl_enter();
  RC_SETUP();
  load_request(c);
  pack_block_pass(c, mask, blk, H, use_target ? st.target + (long long)c.r * S.G : nullptr);
  if (threadIdx.x == 0) {
    *blk.skip = 0;
    *H.skip = 0;
  }
  store_request(c);
}

// full_forward of branch k (all L positions from an empty cache); the head
// slots of branch k report every masked position (slot j <-> position j)
__global__ void k_seam_full_pack(Dims D, Sess S, DevState st, Pass full, Pass blk, Head H, int k, int use_target) {
  pdl_enter();
  RC_SETUP();
  const int r = c.r;
  load_request(c);
  if (threadIdx.x == 0) {
    for (int kk = 0; kk < MAXB; ++kk) {
      full.rng_off[r * MAXB + kk] = r * S.L;
      full.rng_cnt[r * MAXB + kk] = kk == k ? S.L : 0;
    }
    full.n_items[r] = 1;
    int* it = full.items + (long long)r * ITW;
    it[0] = 1 << k;
    it[1] = 0;
    it[2] = S.n_lp;
    it[3] = k;
    for (int lp = 0; lp < S.n_lp; ++lp) c.write_intent(k, lp, false);  // fully rewritten
    *full.skip = 0;
    *H.skip = 0;
  }
  __syncthreads();
  for (int p = threadIdx.x; p < S.L; p += blockDim.x) {
    const int row = r * S.L + p;
    full.slot_pos[row] = p;
    full.slot_req[row] = r;
    full.slot_br[row] = k;
    full.slot_tok[row] = c.rows[k * S.L + p];
    full.slot_kvoff[row] = kv_row_off(D, S, st, r, k, p);
  }
  const int* target = use_target ? st.target + (long long)r * S.G : nullptr;
  for (int j = threadIdx.x; j < S.bs[k]; j += blockDim.x) {
    const int slot = r * S.NRq + S.off[k] + j;
    const bool in = j < S.L && c.rows[k * S.L + j] == c.mask_id;
    blk.slot_req[slot] = r;
    blk.slot_br[slot] = k;
    blk.slot_pos[slot] = in ? j : -1;
    H.masked[slot] = in ? 1 : 0;
    if (in) slot_boost(D, S, c.rows + k * S.L, target, j, &H.boost[slot], &H.tgt[slot]);
    else {
      H.boost[slot] = 0.0f;
      H.tgt[slot] = -1;
    }
  }
}

__global__ void k_step_commit(Dims D, Sess S, DevState st, Pass blk, Head H) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 13);
  RC_SETUP();
  load_request(c);
  if (c.ctrl[C_STATUS] != 0) return;
  __shared__ int s_n, s_ready;
  const int active = c.ctrl[C_ACTIVE_MASK];
  if (threadIdx.x == 0) s_ready = 0;
  for (int k = 0; k < S.B; ++k) {
    if (!((active >> k) & 1)) continue;
    __syncthreads();
    {
      const int nc = apply_commits(c, blk, H, k, S.tau_conf);
      if (threadIdx.x == 0) s_n = nc;
    }
    __syncthreads();
    const int dec = c.count_decoded(k);
    if (threadIdx.x == 0) {
      c.B_(k, B_DEC) = dec;
      c.ctrl[C_COMMITS] += s_n;
      c.emit(EV_DECODE, k, s_n);
    }
    __syncthreads();
    int eos = -1;
    const int st_e = c.check_eos(k, &eos);
    if (st_e == 2) {
      if (threadIdx.x == 0) {
        s_ready |= 1 << k;
        c.emit(EV_EOS_READY, k, eos);
      }
    } else if (st_e == 1) {
      c.realign_for_eos(k);
      if (threadIdx.x == 0) c.emit(EV_EOS_PENDING, k);
    }
    __syncthreads();
  }
  __syncthreads();
  if (s_ready) {
    // select_eos_winner (scheduler.py:216-222): all branches, first max (decoded, -block_size)
    int win = -1;
    for (int k = 0; k < S.B; ++k) {
      const int st_e = c.check_eos(k, nullptr);
      if (st_e != 2) continue;
      if (win < 0 || c.B_(k, B_DEC) > c.B_(win, B_DEC) ||
          (c.B_(k, B_DEC) == c.B_(win, B_DEC) && -c.B_(k, B_SIZE) > -c.B_(win, B_SIZE)))
        win = k;
    }
    const int eos = c.earliest_eos(win);
    if (threadIdx.x == 0) {
      c.emit(EV_FINISH, win, eos);
      c.ctrl[C_WINNER] = win;
      c.ctrl[C_EOS] = eos;
      c.ctrl[C_STATUS] = 1;
    }
  } else {
    for (int k = 0; k < S.B; ++k) c.advance_while_complete(k);
  }
  store_request(c);
}

// ------------------------------------------------------------------ merge
// P_d(i, v) for merge candidates (scheduler.py:180-184 reads dest.prob_map[i, v]).
template <typename T>
__global__ void __launch_bounds__(256) k_merge_prep(Dims D, Sess S, DevState st, const T* __restrict__ head) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 14);
  const int nch = (S.G + 7) / 8;
  const int r = blockIdx.x / (S.B * nch);
  const int d = (blockIdx.x / nch) % S.B;
  const int ch = blockIdx.x % nch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = S.P + ch * 8 + warp;
  if (i >= S.L) return;
  const int* ctrl = st.ctrl + (long long)r * C_WORDS;
  const long long pmi = ((long long)r * S.B + d) * S.L + i;
  uint8_t* ok = st.ptab_ok + pmi;
  const int mask_id = D.V + 1;
  const int* rows = st.tokens + (long long)r * S.B * S.L;
  const int* brs = st.br + (long long)r * S.B * B_WORDS;
  bool need = ctrl[C_STATUS] == 0 && !brs[d * B_WORDS + B_DONE] && rows[d * S.L + i] == mask_id &&
              st.covered[pmi] != 0;
  int cand = 0;
  if (need)
    for (int s = 0; s < S.B; ++s)
      if (s != d && !brs[s * B_WORDS + B_DONE] && rows[s * S.L + i] != mask_id) cand |= 1 << s;
  if (!need || cand == 0) {
    if (lane == 0) *ok = 0;
    return;
  }
  const T* h = reinterpret_cast<const T*>(st.pm_h) + pmi * D.d;
  const T* hl = st.pm_h_lo != nullptr ? reinterpret_cast<const T*>(st.pm_h_lo) + pmi * D.d : nullptr;
  const float m = st.pm_m[pmi], ssum = st.pm_s[pmi], boost = st.pm_boost[pmi];
  const int tg = st.target[(long long)r * S.G + (i - S.P)];
  for (int s = 0; s < S.B; ++s) {
    if (!((cand >> s) & 1)) continue;
    const int v = rows[s * S.L + i];
    const T* w = head + (long long)v * D.d;
    float a = 0.0f;
    constexpr int VE = 16 / sizeof(T);  // elements per 16-byte vector
    for (int c = lane * VE; c < D.d; c += 32 * VE) {
      const uint4 hv = *reinterpret_cast<const uint4*>(h + c), wv = *reinterpret_cast<const uint4*>(w + c);
      const T* hp = reinterpret_cast<const T*>(&hv);
      const T* wp = reinterpret_cast<const T*>(&wv);
#pragma unroll
      for (int e = 0; e < VE; ++e) a = fmaf(ldf(hp + e), ldf(wp + e), a);
      if (hl != nullptr) {  // bf16x2: the head input's lo plane (the head GEMM used h_hi + h_lo)
        const uint4 lv = *reinterpret_cast<const uint4*>(hl + c);
        const T* lp = reinterpret_cast<const T*>(&lv);
#pragma unroll
        for (int e = 0; e < VE; ++e) a = fmaf(ldf(lp + e), ldf(wp + e), a);
      }
    }
    a = warp_sum(a);
    float l = head_logit(a, D.head_scale, D.spike_cut, D.spike_gain);
    if (v == tg && tg <= D.V) l += boost;
    if (lane == 0) st.ptab[pmi * S.B + s] = expf(l - m) / ssum;
  }
  if (lane == 0) *ok = 1;
}

// probability lookup for (dest d, pos i, token v) from the prep table; thread 0
__device__ float merge_prob(RC& c, int d, int i, int v) {
  const long long pmi = ((long long)c.r * c.S->B + d) * c.S->L + i;
  if (!c.st.ptab_ok[pmi]) {
    c.ctrl[C_STATUS] = BB_ERR_STATE;
    return 0.0f;
  }
  const int* g = c.st.tokens + (long long)c.r * c.S->B * c.S->L;
  const int* gb = c.st.br + (long long)c.r * c.S->B * B_WORDS;
  for (int s = 0; s < c.S->B; ++s)
    if (s != d && !gb[s * B_WORDS + B_DONE] && g[s * c.S->L + i] == v) return c.st.ptab[pmi * c.S->B + s];
  c.ctrl[C_STATUS] = BB_ERR_STATE;
  return 0.0f;
}

// Alg. 2 (scheduler.py:144-209).  `cov` = smem covered flags [B][L].
__device__ void merge_sync_core(RC& c, uint8_t* cov, bool copy_device_state, int* mfill, float* mpv,
                                const float* mprob) {
  const Sess& S = *c.S;
  __shared__ int s_order[MAXB], s_srcs, s_leader, s_parts;
  int ld = c.leader();
  if (c.B_(ld, B_DEC) == 0) return;
  if (threadIdx.x == 0) {
    int parts = 0;
    for (int k = 0; k < S.B; ++k)
      if (!c.B_(k, B_DONE)) parts |= 1 << k;
    s_parts = parts;
    // dest order: ascending (tokens_decoded, index)
    int n = 0;
    for (int k = 0; k < S.B; ++k)
      if ((parts >> k) & 1) s_order[n++] = k;
    for (int a = 1; a < n; ++a)
      for (int b = a; b > 0; --b) {
        const int x = s_order[b - 1], y = s_order[b];
        if (c.B_(y, B_DEC) < c.B_(x, B_DEC) || (c.B_(y, B_DEC) == c.B_(x, B_DEC) && y < x)) {
          s_order[b - 1] = y;
          s_order[b] = x;
        } else break;
      }
    for (int a = n; a < MAXB; ++a) s_order[a] = -1;
  }
  __syncthreads();
  const int parts = s_parts;
  if (S.merge_en) {
    for (int oi = 0; oi < MAXB; ++oi) {
      const int d = s_order[oi];
      if (d < 0) break;
      if (threadIdx.x == 0) s_srcs = 0;
      __syncthreads();
      for (int s = 0; s < S.B; ++s) {
        if (s == d || !((parts >> s) & 1)) continue;
        const bool ok = c.compatible(d, s);
        if (ok && threadIdx.x == 0) s_srcs |= 1 << s;
        __syncthreads();
      }
      const int srcs = s_srcs;
      if (srcs) {
        // positions of the union of the sources' windows are independent for one
        // destination (a fill only changes drow[i]): evaluate them in parallel,
        // then apply fills / emit events in position order.
        __shared__ int s_lo, s_hi;
        if (threadIdx.x == 0) {
          int lo = S.L, hi = 0;
          for (int s2 = 0; s2 < S.B; ++s2)
            if ((srcs >> s2) & 1) {
              lo = min(lo, c.B_(s2, B_START));
              hi = max(hi, c.B_(s2, B_END));
            }
          s_lo = lo;
          s_hi = hi;
        }
        __syncthreads();
        const int lo = s_lo, hi = s_hi;
        int* rd = c.row(d);
        for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
          int best = -1;
          float bp = 0.0f;
          bool in_union = false;
          for (int s2 = 0; s2 < S.B; ++s2)
            if (((srcs >> s2) & 1) && c.B_(s2, B_START) <= i && i < c.B_(s2, B_END)) in_union = true;
          if (in_union && rd[i] == c.mask_id && cov[d * S.L + i]) {
            for (int s2 = 0; s2 < S.B; ++s2) {
              if (!((srcs >> s2) & 1)) continue;
              const int v = c.row(s2)[i];
              if (v == c.mask_id) continue;
              const float p = mprob ? mprob[((long long)d * S.L + i) * S.B + s2] : merge_prob(c, d, i, v);
              if (best < 0 || p > bp) {
                best = s2;
                bp = p;
              }
            }
          }
          mfill[i] = (best >= 0 && bp > S.tau_merge) ? best : -1;
          mpv[i] = bp;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          for (int i = lo; i < hi; ++i) {
            const int best = mfill[i];
            if (best < 0) continue;
            const int tok = c.row(best)[i];
            rd[i] = tok;
            c.B_(d, B_MERGED) += 1;
            c.B_(d, B_DEC) += 1;  // i >= P: one gen mask became a token
            c.ctrl[C_MERGES] += 1;
            c.emit(EV_MERGE, d, best, i, tok, 0, mpv[i]);
          }
        }
      }
      __syncthreads();
      c.advance_while_complete(d);
    }
  }
  if (S.sync_en) {
    if (threadIdx.x == 0) s_leader = c.leader();
    __syncthreads();
    const int L_ = s_leader;
    for (int d = 0; d < S.B; ++d) {
      if (!((parts >> d) & 1) || d == L_ || c.B_(d, B_DONE)) continue;
      const int gap = c.B_(L_, B_DEC) - c.B_(d, B_DEC);
      if (!((float)gap > S.tau_sync)) continue;
      int* rd = c.row(d);
      const int* rl = c.row(L_);
      for (int i = threadIdx.x; i < S.L; i += blockDim.x) {
        rd[i] = rl[i];
        cov[d * S.L + i] = cov[L_ * S.L + i];
      }
      if (copy_device_state) {
        const long long bd = ((long long)c.r * S.B + d) * S.L, bl = ((long long)c.r * S.B + L_) * S.L;
        for (int i = threadIdx.x; i < S.L; i += blockDim.x) {
          c.st.pm_m[bd + i] = c.st.pm_m[bl + i];
          c.st.pm_s[bd + i] = c.st.pm_s[bl + i];
          c.st.pm_boost[bd + i] = c.st.pm_boost[bl + i];
        }
      }
      __syncthreads();
      if (threadIdx.x == 0 && copy_device_state) {
        // KV: alias the leader's pages (copy-on-write later)
        int* td = c.pt(d);
        const int* tl = c.pt(L_);
        for (int lp = 0; lp < S.n_lp; ++lp) {
          const int old = td[lp];
          td[lp] = tl[lp];
          c.refc()[tl[lp]] += 1;
          c.pg_decref(old);
        }
        const int n = c.ctrl[C_NPMCOPY];
        if (n < MAXB) {
          c.st.pm_copies[((long long)c.r * MAXB + n) * 2] = L_;
          c.st.pm_copies[((long long)c.r * MAXB + n) * 2 + 1] = d;
          c.ctrl[C_NPMCOPY] = n + 1;
        }
      }
      c.realign_to_first_mask(d);
      const int dec = c.count_decoded(d);
      if (threadIdx.x == 0) {
        c.B_(d, B_DEC) = dec;
        c.ctrl[C_SYNCS] += 1;
        c.emit(EV_SYNC, d, L_, gap);
      }
      __syncthreads();
    }
  }
}

__global__ void k_merge_sync(Dims D, Sess S, DevState st, int after_prefill) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 15);
  RC_SETUP();
  load_request(c);
  if (c.ctrl[C_STATUS] != 0) return;
  uint8_t* cov = reinterpret_cast<uint8_t*>(c.rows + S.B * S.L);
  const long long cb = (long long)c.r * S.B * S.L;
  for (int i = threadIdx.x; i < S.B * S.L; i += blockDim.x) cov[i] = st.covered[cb + i];
  __shared__ int s_ev0;
  if (threadIdx.x == 0) {
    c.ctrl[C_NPMCOPY] = 0;
    s_ev0 = c.ctrl[C_NEV];
  }
  __syncthreads();
  int* mfill = reinterpret_cast<int*>(cov + ((S.B * S.L + 15) & ~15));
  merge_sync_core(c, cov, true, mfill, reinterpret_cast<float*>(mfill + S.L), nullptr);
  __syncthreads();
  // scheduler.py:370-372 emits merge/sync events after merge_sync returns:
  // their `decoded` snapshot is the post-merge/sync state.
  if (threadIdx.x == 0 && S.trace) {
    const int n1 = min(c.ctrl[C_NEV], S.ev_cap);
    for (int n = s_ev0; n < n1; ++n) {
      int* e = st.events + ((long long)c.r * S.ev_cap + n) * EVW;
      for (int k = 0; k < S.B; ++k) e[E_DEC + k] = c.B_(k, B_DEC);
    }
  }
  for (int i = threadIdx.x; i < S.B * S.L; i += blockDim.x) st.covered[cb + i] = cov[i];
  if (threadIdx.x == 0) {
    bool any_live = false;
    for (int k = 0; k < S.B; ++k) any_live |= !c.B_(k, B_DONE);
    if (!after_prefill && c.ctrl[C_SINCE_REFRESH] >= S.refresh_interval) {
      int m = 0;
      for (int k = 0; k < S.B; ++k)
        if (!c.B_(k, B_DONE)) m |= 1 << k;
      c.ctrl[C_REFRESH_MASK] = m;
      if (m) c.ctrl[C_REFRESH_DUE] = 1;
      else c.ctrl[C_SINCE_REFRESH] = 0;
    }
    c.ctrl[C_WINNER] = -1;
  }
  __syncthreads();
  bool all_done = true;
  for (int k = 0; k < S.B; ++k) all_done &= c.B_(k, B_DONE) != 0;
  if (all_done) {
    // final selection (scheduler.py:393-394)
    int win = 0;
    for (int k = 1; k < S.B; ++k)
      if (c.B_(k, B_DEC) > c.B_(win, B_DEC) ||
          (c.B_(k, B_DEC) == c.B_(win, B_DEC) && -c.B_(k, B_SIZE) > -c.B_(win, B_SIZE)))
        win = k;
    const int eos = c.earliest_eos(win);
    if (threadIdx.x == 0) {
      c.emit(EV_FINISH, win, eos);
      c.ctrl[C_WINNER] = win;
      c.ctrl[C_EOS] = eos;
      c.ctrl[C_STATUS] = 1;
    }
  }
  store_request(c);
}

// ------------------------------------------------------------------ refresh
// k >= 0: branch k's full pass (rows r * L + p); k = -1: every refreshing
// branch stacked into one pass (full.nseq = B; branch kk at rows
// (r * B + kk) * L + p, its own key list).  The page allocations run in the
// same branch order either way, so both give the same page tables.
__global__ void k_refresh_pack(Dims D, Sess S, DevState st, Pass full, Pass blk, Head H, int k) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 16);
  RC_SETUP();
  const int r = c.r;
  load_request(c);
  const bool due = c.ctrl[C_STATUS] == 0 && c.ctrl[C_REFRESH_DUE];
  const int rmask = c.ctrl[C_REFRESH_MASK];
  const int k0 = k < 0 ? 0 : k, k1 = k < 0 ? S.B : k + 1;
  auto live_of = [&](int kk) { return due && ((rmask >> kk) & 1) && kk >= k0 && kk < k1; };
  auto group_of = [&](int kk) { return r * full.nseq + (k < 0 ? kk : 0); };
  if (threadIdx.x == 0) {
    int nl = 0;
    for (int kk = 0; kk < MAXB; ++kk) {
      const bool lv = kk < S.B && live_of(kk);
      full.rng_off[r * MAXB + kk] = (kk < S.B ? group_of(kk) : r * full.nseq) * S.L;
      full.rng_cnt[r * MAXB + kk] = lv ? S.L : 0;
      nl += lv ? 1 : 0;
    }
    // planned attention items (SIMT path): one per-branch pass only
    full.n_items[r] = (k >= 0 && nl) ? 1 : 0;
    if (k >= 0 && nl) {
      int* it = full.items + (long long)r * ITW;
      it[0] = 1 << k;
      it[1] = 0;
      it[2] = S.n_lp;
      it[3] = k;
    }
    for (int kk = k0; kk < k1; ++kk)
      if (live_of(kk))
        for (int lp = 0; lp < S.n_lp; ++lp) c.write_intent(kk, lp, false);  // fully rewritten
    if (nl) {
      *full.skip = 0;
      *H.skip = 0;
    }
  }
  __syncthreads();
  for (int kk = k0; kk < k1; ++kk) {
    const bool live = live_of(kk);
    const int g = group_of(kk);
    for (int p = threadIdx.x; p < S.L; p += blockDim.x) {
      const int row = g * S.L + p;
      full.slot_pos[row] = live ? p : -1;
      full.slot_req[row] = r;
      full.slot_br[row] = kk;
      full.slot_tok[row] = c.rows[kk * S.L + p];
      full.slot_kvoff[row] = live ? kv_row_off(D, S, st, r, kk, p) : 0;
    }
    const int* target = st.target + (long long)r * S.G;
    const int rbase = blk_base(S, blk, r);
    for (int j = threadIdx.x; j < S.bs[kk] && rbase >= 0; j += blockDim.x) {
      const int slot = rbase + S.off[kk] + j;
      const int pos = c.B_(kk, B_START) + j;
      const bool in = live && pos < c.B_(kk, B_END) && c.rows[kk * S.L + pos] == c.mask_id;
      blk.slot_req[slot] = r;
      blk.slot_br[slot] = kk;
      blk.slot_pos[slot] = in ? pos : -1;
      H.masked[slot] = in ? 1 : 0;
      if (in) slot_boost(D, S, c.rows + kk * S.L, target, pos, &H.boost[slot], &H.tgt[slot]);
      else {
        H.boost[slot] = 0.0f;
        H.tgt[slot] = -1;
      }
    }
  }
}

__global__ void k_refresh_end(Dims D, Sess S, DevState st) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 17);
  RC_SETUP();
  load_request(c);
  if (threadIdx.x == 0 && c.ctrl[C_STATUS] == 0 && c.ctrl[C_REFRESH_DUE]) {
    c.ctrl[C_NFE2] += 1;
    c.ctrl[C_REFRESHES] += 1;
    c.emit(EV_REFRESH, -1, c.ctrl[C_REFRESH_MASK]);
    c.ctrl[C_SINCE_REFRESH] = 0;
    c.ctrl[C_REFRESH_DUE] = 0;
  }
}

// ------------------------------------------------------------------ vanilla decode
// decoding.py:279-321, the baseline decoder of SURVEY 8(f3): one FULL forward
// per round over the whole row (no cache reuse), then Eq. 1 with tau = 1.0 over
// the masked positions of [P, first eos or L) -- the most confident position
// commits -- charged as nfe_block.  The session has one branch of block size G,
// so its G head slots cover the span.  k_prefill_init sets the initial state;
// each round: k_vanilla_pack -> full pass of branch 0 -> head -> k_vanilla_commit.
__global__ void k_vanilla_pack(Dims D, Sess S, DevState st, Pass full, Pass blk, Head H) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 19);
  RC_SETUP();
  const int r = c.r;
  __shared__ int s_live;
  load_request(c);
  if (threadIdx.x == 0) {
    s_live = c.ctrl[C_STATUS] == 0;
    if (s_live) {
      c.ctrl[C_ITER] += 1;
      const int total = c.ctrl[C_NFE0] + c.ctrl[C_NFE1] + c.ctrl[C_NFE2];
      if (total > S.hard_cap) {  // decoding.py:296-297
        c.ctrl[C_STATUS] = BB_ERR_RUNAWAY;
        s_live = 0;
      }
    }
  }
  __syncthreads();
  int end = S.L;
  bool any = false;
  if (s_live) {
    const int eos = c.earliest_eos(0);
    end = eos >= 0 ? eos : S.L;
    any = c.has_mask(0, S.P, end);
    if (!any) {  // no mask before the first eos: finished (decoding.py:302-305, 317-321)
      const int dec = c.count_decoded(0);
      if (threadIdx.x == 0) {
        c.B_(0, B_DEC) = dec;
        c.emit(EV_FINISH, 0, eos);
        c.ctrl[C_WINNER] = 0;
        c.ctrl[C_EOS] = eos;
        c.ctrl[C_STATUS] = 1;
      }
    }
  }
  __syncthreads();
  const bool live = s_live && any;
  if (threadIdx.x == 0) {
    c.B_(0, B_START) = S.P;
    c.B_(0, B_END) = end;
    for (int kk = 0; kk < MAXB; ++kk) {
      full.rng_off[r * MAXB + kk] = r * S.L;
      full.rng_cnt[r * MAXB + kk] = (live && kk == 0) ? S.L : 0;
    }
    full.n_items[r] = live ? 1 : 0;
    if (live) {
      int* it = full.items + (long long)r * ITW;
      it[0] = 1;
      it[1] = 0;
      it[2] = S.n_lp;
      it[3] = 0;
      *full.skip = 0;
      *H.skip = 0;
    }
  }
  __syncthreads();
  for (int p = threadIdx.x; p < S.L; p += blockDim.x) {
    const int row = r * S.L + p;
    full.slot_pos[row] = live ? p : -1;
    full.slot_req[row] = r;
    full.slot_br[row] = 0;
    full.slot_tok[row] = c.rows[p];
    full.slot_kvoff[row] = live ? kv_row_off(D, S, st, r, 0, p) : 0;
  }
  const int* target = st.target + (long long)r * S.G;
  const int vbase = blk_base(S, blk, r);
  for (int j = threadIdx.x; j < S.NRq && vbase >= 0; j += blockDim.x) {
    const int slot = vbase + j;
    const int pos = S.P + j;
    const bool in = live && pos < end && c.rows[pos] == c.mask_id;
    blk.slot_req[slot] = r;
    blk.slot_br[slot] = 0;
    blk.slot_pos[slot] = in ? pos : -1;
    H.masked[slot] = in ? 1 : 0;
    if (in) slot_boost(D, S, c.rows, target, pos, &H.boost[slot], &H.tgt[slot]);
    else {
      H.boost[slot] = 0.0f;
      H.tgt[slot] = -1;
    }
  }
  store_request(c);
}

__global__ void k_vanilla_commit(Dims D, Sess S, DevState st, Pass blk, Head H) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 13);
  RC_SETUP();
  load_request(c);
  __shared__ int s_live;
  if (threadIdx.x == 0) s_live = c.ctrl[C_STATUS] == 0 && c.B_(0, B_END) > S.P && *H.skip == 0;
  __syncthreads();
  if (!s_live) return;
  // only this request's slots are masked when its round is live
  bool any = false;
  const int vbase = blk_base(S, blk, c.r);
  for (int j = threadIdx.x; j < S.NRq && vbase >= 0; j += blockDim.x) any |= H.masked[vbase + j] != 0;
  if (!__syncthreads_or(any)) return;
  const int n = apply_commits(c, blk, H, 0, 1.0f);  // tau 1.0: the most confident position (decoding.py:311)
  const int dec = c.count_decoded(0);
  if (threadIdx.x == 0) {
    c.B_(0, B_DEC) = dec;
    c.ctrl[C_NFE1] += 1;
    c.ctrl[C_COMMITS] += n;
    c.emit(EV_BLOCK, 0, 1);
  }
  store_request(c);
}

// ------------------------------------------------------------------ KV-space diagnostics
// kv_vectorize (model.py:346-352) of (request r, branch k): fp32
// [layers][L][2][kv_dim], keys before values; CTA per (position, layer).
template <typename T>
__global__ void __launch_bounds__(256) k_kv_gather(Dims D, Sess S, DevState st, int r, int k, float* dst) {
  pdl_enter();
  const int pos = blockIdx.x, l = blockIdx.y;
  const int kv_dim = D.nkv * D.hd;
  const int lp = lp_of(S, pos);
  const long long gpage = (long long)r * S.pool + st.pt[((long long)r * S.B + k) * S.n_lp + lp];
  const long long lay = (long long)l * S.R * S.pool * D.nkv * S.ps * D.hd;
  const int row = pos - lp_start(S, lp);
  float* o = dst + ((long long)l * S.L + pos) * 2 * kv_dim;
  for (int e = threadIdx.x; e < kv_dim; e += blockDim.x) {
    const int kvh = e / D.hd, i = e - kvh * D.hd;
    const long long src = lay + ((gpage * D.nkv + kvh) * S.ps + row) * D.hd + i;
    const T* kp = reinterpret_cast<const T*>(st.kv_k) + src;
    const T* vp = reinterpret_cast<const T*>(st.kv_v) + src;
    // bf16x2: the cached value is hi + lo
    o[e] = ldf(kp) + (st.kv_lo != 0 ? ldf(kp + st.kv_lo) : 0.0f);
    o[kv_dim + e] = ldf(vp) + (st.kv_lo != 0 ? ldf(vp + st.kv_lo) : 0.0f);
  }
}

// inverse of k_kv_gather: a dense kv_vectorize-layout cache -> branch k's
// pages (rounded to the model dtype); the seams' cache upload
template <typename T>
__global__ void __launch_bounds__(256) k_kv_scatter(Dims D, Sess S, DevState st, int r, int k, const float* src) {
  pdl_enter();
  const int pos = blockIdx.x, l = blockIdx.y;
  const int kv_dim = D.nkv * D.hd;
  const int lp = lp_of(S, pos);
  const long long gpage = (long long)r * S.pool + st.pt[((long long)r * S.B + k) * S.n_lp + lp];
  const long long lay = (long long)l * S.R * S.pool * D.nkv * S.ps * D.hd;
  const int row = pos - lp_start(S, lp);
  const float* o = src + ((long long)l * S.L + pos) * 2 * kv_dim;
  for (int e = threadIdx.x; e < kv_dim; e += blockDim.x) {
    const int kvh = e / D.hd, i = e - kvh * D.hd;
    const long long dst = lay + ((gpage * D.nkv + kvh) * S.ps + row) * D.hd + i;
    T* kp = reinterpret_cast<T*>(st.kv_k) + dst;
    T* vp = reinterpret_cast<T*>(st.kv_v) + dst;
    stf2(kp, st.kv_lo != 0 ? kp + st.kv_lo : nullptr, o[e]);
    stf2(vp, st.kv_lo != 0 ? vp + st.kv_lo : nullptr, o[kv_dim + e]);
  }
}

// Point branch k of request r at the reserved scratch pages (saving its page
// table) and set the full pass up for that one row (the other requests' rows
// are padding).  CTA per request.
__global__ void k_fresh_pack(Dims D, Sess S, DevState st, Pass full, int r, int k, int* save) {
  pdl_enter();
  const int rr = blockIdx.x;
  const bool live = rr == r;
  int* pt = st.pt + ((long long)rr * S.B + k) * S.n_lp;
  if (live)
    for (int lp = threadIdx.x; lp < S.n_lp; lp += blockDim.x) {
      save[lp] = pt[lp];
      pt[lp] = S.pool - S.n_lp + lp;
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int kk = 0; kk < MAXB; ++kk) {
      full.rng_off[rr * MAXB + kk] = rr * S.L;
      full.rng_cnt[rr * MAXB + kk] = (live && kk == k) ? S.L : 0;
    }
    full.n_items[rr] = live ? 1 : 0;
    if (live) {
      int* it = full.items + (long long)rr * ITW;
      it[0] = 1 << k;
      it[1] = 0;
      it[2] = S.n_lp;
      it[3] = k;
      *full.skip = 0;
    }
  }
  const int* rw = st.tokens + ((long long)rr * S.B + k) * S.L;
  for (int p = threadIdx.x; p < S.L; p += blockDim.x) {
    const int row = rr * S.L + p;
    full.slot_pos[row] = live ? p : -1;
    full.slot_req[row] = rr;
    full.slot_br[row] = k;
    full.slot_tok[row] = rw[p];
    full.slot_kvoff[row] = live ? kv_row_off(D, S, st, rr, k, p) : 0;
  }
}

__global__ void k_fresh_restore(Sess S, DevState st, int r, int k, const int* save) {
  pdl_enter();
  int* pt = st.pt + ((long long)r * S.B + k) * S.n_lp;
  for (int lp = threadIdx.x; lp < S.n_lp; lp += blockDim.x) pt[lp] = save[lp];
}

// ||a - b||_2 in fp64: per-CTA strided partial sums, then one ordered sum
__global__ void __launch_bounds__(256) k_sqdiff_partial(const float* a, const float* b, long long n, double* part) {
  pdl_enter();
  __shared__ double sh[256];
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double d = (double)a[i] - (b != nullptr ? (double)b[i] : 0.0);
    acc += d * d;
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x >> 1; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void k_sqdiff_final(const double* part, int n, double* out) {
  pdl_enter();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    out[0] = sqrt(s);
  }
}

// ------------------------------------------------------------------ copies
// 16-byte vector copies; block-strided over (request, job, layer) units.
template <typename T>
__global__ void __launch_bounds__(512) k_copy_pages(Dims D, Sess S, DevState st, int with_pm) {
  pdl_enter();
  klog_mark(D.klog, D.klog_cap, 18);
  if (!with_pm) {
    const long long vecs = (long long)D.nkv * S.ps * D.hd * sizeof(T) / 16;  // per (page, layer)
    __shared__ int s_any;
    if (threadIdx.x == 0) {
      int a = 0;
      for (int r = 0; r < S.R && !a; ++r) a = st.ctrl[(long long)r * C_WORDS + C_NCOPY] > 0;
      s_any = a;
    }
    __syncthreads();
    if (!s_any) return;
    const long long units = (long long)S.R * S.max_copies * D.layers;
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
      const int layer = (int)(u % D.layers);
      const int j = (int)((u / D.layers) % S.max_copies);
      const int r = (int)(u / ((long long)D.layers * S.max_copies));
      if (j >= st.ctrl[(long long)r * C_WORDS + C_NCOPY]) continue;
      const int src = st.copies[((long long)r * S.max_copies + j) * 2];
      const int dst = st.copies[((long long)r * S.max_copies + j) * 2 + 1];
      const long long lay = (long long)layer * S.R * S.pool;
      const long long so = (lay + (long long)r * S.pool + src) * vecs, dof = (lay + (long long)r * S.pool + dst) * vecs;
      uint4* K = reinterpret_cast<uint4*>(st.kv_k);
      uint4* V = reinterpret_cast<uint4*>(st.kv_v);
      for (long long e = threadIdx.x; e < vecs; e += blockDim.x) {
        const uint4 a = K[so + e], b = V[so + e];
        K[dof + e] = a;
        V[dof + e] = b;
      }
      if (st.kv_lo != 0) {  // bf16x2: the lo pools (kv_lo elements on)
        const long long lo = st.kv_lo * (long long)sizeof(T) / 16;
        for (long long e = threadIdx.x; e < vecs; e += blockDim.x) {
          const uint4 a = K[lo + so + e], b = V[lo + so + e];
          K[lo + dof + e] = a;
          V[lo + dof + e] = b;
        }
      }
    }
  } else {
    const int vecs = (int)(D.d * sizeof(T) / 16);
    __shared__ int s_any;
    if (threadIdx.x == 0) {
      int a = 0;
      for (int r = 0; r < S.R && !a; ++r) a = st.ctrl[(long long)r * C_WORDS + C_NPMCOPY] > 0;
      s_any = a;
    }
    __syncthreads();
    if (!s_any) return;
    // (request, job, position) units
    const long long total = (long long)S.R * MAXB * S.L;
    for (long long u = blockIdx.x; u < total; u += gridDim.x) {
      const int pos = (int)(u % S.L);
      const int j = (int)((u / S.L) % MAXB);
      const int r = (int)(u / ((long long)S.L * MAXB));
      if (j >= st.ctrl[(long long)r * C_WORDS + C_NPMCOPY]) continue;
      const int src = st.pm_copies[((long long)r * MAXB + j) * 2];
      const int dst = st.pm_copies[((long long)r * MAXB + j) * 2 + 1];
      const uint4* a = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(st.pm_h) +
                                                      (((long long)r * S.B + src) * S.L + pos) * D.d);
      uint4* b = reinterpret_cast<uint4*>(reinterpret_cast<T*>(st.pm_h) + (((long long)r * S.B + dst) * S.L + pos) * D.d);
      for (int e = threadIdx.x; e < vecs; e += blockDim.x) b[e] = a[e];
      if (st.pm_h_lo != nullptr) {
        const uint4* al = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(st.pm_h_lo) +
                                                         (((long long)r * S.B + src) * S.L + pos) * D.d);
        uint4* bl = reinterpret_cast<uint4*>(reinterpret_cast<T*>(st.pm_h_lo) +
                                             (((long long)r * S.B + dst) * S.L + pos) * D.d);
        for (int e = threadIdx.x; e < vecs; e += blockDim.x) bl[e] = al[e];
      }
    }
  }
}

// ------------------------------------------------------------------ launch helpers
static size_t rc_smem(const Sess& S) { return (size_t)S.B * S.L * 4 + (size_t)S.B * S.L + 16 + (size_t)S.L * 8 + 64; }

template <typename K>
static void big_smem(K kern) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

// ------------------------------------------------------------------ kernel-level seams
// confidence_transition on given probabilities (decoding.py:108-129).
__global__ void k_debug_commit(const float* probs, int n, int n_out, const int* pos, int* row, float tau, int* out,
                               int* count) {
  pdl_enter();
  extern __shared__ float sconf[];
  int* sarg = reinterpret_cast<int*>(sconf + n);
  int* sval = sarg + n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < n; j += blockDim.x >> 5) {
    float m = -INFINITY;
    int a = 0x7fffffff;
    for (int v = lane; v < n_out; v += 32) {
      const float x = probs[(long long)j * n_out + v];
      if (x > m) {
        m = x;
        a = v;
      }
    }
    warp_argmax(m, a);
    if (lane == 0) {
      sconf[j] = m;
      sarg[j] = a;
      sval[j] = 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *count = eq1_commit(sconf, sarg, pos, sval, n, tau, row, out);
}

// merge_sync on given rows / branch states / full probability maps
// (scheduler.py:144-209): the production merge core, fed from a table built
// out of the caller's prob maps instead of the stored head rows.
__global__ void k_debug_merge(Dims D, Sess S, DevState st, const float* probmaps, int n_out) {
  pdl_enter();
  RC_SETUP();
  const int mask_id = D.V + 1;
  for (int idx = threadIdx.x; idx < S.B * S.L; idx += blockDim.x) {
    const int d = idx / S.L, i = idx % S.L;
    for (int s2 = 0; s2 < S.B; ++s2) {
      const int v = st.tokens[s2 * S.L + i];
      st.ptab[(long long)idx * S.B + s2] = v != mask_id ? probmaps[(long long)idx * n_out + v] : 0.0f;
    }
    st.ptab_ok[idx] = 1;
    (void)d;
  }
  __syncthreads();
  load_request(c);
  uint8_t* cov = reinterpret_cast<uint8_t*>(c.rows + S.B * S.L);
  for (int i = threadIdx.x; i < S.B * S.L; i += blockDim.x) cov[i] = st.covered[i];
  __syncthreads();
  int* mfill = reinterpret_cast<int*>(cov + ((S.B * S.L + 15) & ~15));
  merge_sync_core(c, cov, false, mfill, reinterpret_cast<float*>(mfill + S.L), nullptr);
  __syncthreads();
  for (int i = threadIdx.x; i < S.B * S.L; i += blockDim.x) st.covered[i] = cov[i];
  store_request(c);
}

cudaError_t launch_debug_commit(const float* probs, int n, int n_out, const int* pos, int* row, float tau, int* out,
                                int* count, cudaStream_t s) {
  launch_k(k_debug_commit, dim3(1), dim3(256), (size_t)((size_t)n * 12 + 16), s, probs, n, n_out, pos, row, tau, out, count);
  return cudaGetLastError();
}
cudaError_t launch_debug_merge(const Dims& D, const Sess& S, const DevState& st, const float* probmaps, int n_out,
                               cudaStream_t s) {
  static bool a = false;
  if (!a) {
    big_smem(k_debug_merge);
    a = true;
  }
  launch_k(k_debug_merge, dim3(1), dim3(256), (size_t)(rc_smem(S)), s, D, S, st, probmaps, n_out);
  return cudaGetLastError();
}

cudaError_t launch_prefill_init(const Dims& D, const Sess& S, const DevState& st, const Pass& full, const Pass& blk,
                                const Head& H, cudaStream_t s) {
  static bool a = false;
  if (!a) {
    big_smem(k_prefill_init);
    a = true;
  }
  launch_k(k_prefill_init, dim3(S.R), dim3(256), (size_t)(rc_smem(S)), s, D, S, st, full, blk, H);
  return cudaGetLastError();
}
cudaError_t launch_prefill_post(const Dims& D, const Sess& S, const DevState& st, const Pass& blk, const Head& H,
                                cudaStream_t s) {
  static bool a = false;
  if (!a) {
    big_smem(k_prefill_post);
    a = true;
  }
  launch_k(k_prefill_post, dim3(S.R), dim3(256), (size_t)(rc_smem(S)), s, D, S, st, blk, H);
  return cudaGetLastError();
}
cudaError_t launch_block_bases(const Dims& D, const Sess& S, const DevState& st, const Pass& blk, const Head& H,
                               cudaStream_t s) {
  launch_k(k_block_bases, dim3(1), dim3(256), (size_t)0, s, D, S, st, blk, H);
  return cudaGetLastError();
}
cudaError_t launch_block_pack(const Dims& D, const Sess& S, const DevState& st, const Pass& blk, const Head& H,
                              cudaStream_t s) {
  static bool a = false;
  if (!a) {
    big_smem(k_block_pack);
    a = true;
  }
  launch_k(k_block_pack, dim3(S.R), dim3(256), (size_t)(rc_smem(S)), s, D, S, st, blk, H);
  return cudaGetLastError();
}
cudaError_t launch_seam_init(const Dims& D, const Sess& S, const DevState& st, cudaStream_t s) {
  launch_k(k_seam_init, dim3(S.R), dim3(256), (size_t)0, s, D, S, st);
  return cudaGetLastError();
}

cudaError_t launch_seam_block_pack(const Dims& D, const Sess& S, const DevState& st, const Pass& blk, const Head& H,
                                   int mask, int use_target, cudaStream_t s) {
  big_smem(k_seam_block_pack);
  launch_k(k_seam_block_pack, dim3(S.R), dim3(256), rc_smem(S), s, D, S, st, blk, H, mask, use_target);
  return cudaGetLastError();
}

cudaError_t launch_seam_full_pack(const Dims& D, const Sess& S, const DevState& st, const Pass& full, const Pass& blk,
                                  const Head& H, int k, int use_target, cudaStream_t s) {
  big_smem(k_seam_full_pack);
  launch_k(k_seam_full_pack, dim3(S.R), dim3(256), rc_smem(S), s, D, S, st, full, blk, H, k, use_target);
  return cudaGetLastError();
}

cudaError_t launch_copy_pages(const Dims& D, const Sess& S, const DevState& st, int with_pm, cudaStream_t s) {
  if (D.dtype == 1) launch_k(k_copy_pages<__nv_bfloat16>, dim3(2 * S.n_sms), dim3(512), (size_t)(0), s, D, S, st, with_pm);
  else launch_k(k_copy_pages<float>, dim3(2 * S.n_sms), dim3(512), (size_t)(0), s, D, S, st, with_pm);
  return cudaGetLastError();
}
cudaError_t launch_step_commit(const Dims& D, const Sess& S, const DevState& st, const Pass& blk, const Head& H,
                               cudaStream_t s) {
  static bool a = false;
  if (!a) {
    big_smem(k_step_commit);
    a = true;
  }
  launch_k(k_step_commit, dim3(S.R), dim3(256), (size_t)(rc_smem(S)), s, D, S, st, blk, H);
  return cudaGetLastError();
}
cudaError_t launch_merge_prep(const Dims& D, const Sess& S, const DevState& st, const Weights& W, cudaStream_t s) {
  const int nch = (S.G + 7) / 8;
  if (D.dtype == 1) launch_k(k_merge_prep<__nv_bfloat16>, dim3(S.R * S.B * nch), dim3(256), (size_t)(0), s, D, S, st, (const __nv_bfloat16*)W.head);
  else launch_k(k_merge_prep<float>, dim3(S.R * S.B * nch), dim3(256), (size_t)(0), s, D, S, st, (const float*)W.head);
  return cudaGetLastError();
}
cudaError_t launch_merge_sync(const Dims& D, const Sess& S, const DevState& st, int after_prefill, cudaStream_t s) {
  static bool a = false;
  if (!a) {
    big_smem(k_merge_sync);
    a = true;
  }
  launch_k(k_merge_sync, dim3(S.R), dim3(256), (size_t)(rc_smem(S)), s, D, S, st, after_prefill);
  return cudaGetLastError();
}
cudaError_t launch_refresh_begin(const Dims&, const Sess&, const DevState&, const Pass&, const Head&, cudaStream_t) {
  return cudaSuccess;
}
cudaError_t launch_refresh_pack(const Dims& D, const Sess& S, const DevState& st, const Pass& full, const Pass& blk,
                                const Head& H, int branch, cudaStream_t s) {
  static bool a = false;
  if (!a) {
    big_smem(k_refresh_pack);
    a = true;
  }
  launch_k(k_refresh_pack, dim3(S.R), dim3(256), (size_t)(rc_smem(S)), s, D, S, st, full, blk, H, branch);
  return cudaGetLastError();
}
cudaError_t launch_refresh_end(const Dims& D, const Sess& S, const DevState& st, cudaStream_t s) {
  static bool a = false;
  if (!a) {
    big_smem(k_refresh_end);
    a = true;
  }
  launch_k(k_refresh_end, dim3(S.R), dim3(256), (size_t)(rc_smem(S)), s, D, S, st);
  return cudaGetLastError();
}

cudaError_t launch_vanilla_pack(const Dims& D, const Sess& S, const DevState& st, const Pass& full, const Pass& blk,
                                const Head& H, cudaStream_t s) {
  static bool a = false;
  if (!a) {
    big_smem(k_vanilla_pack);
    a = true;
  }
  launch_k(k_vanilla_pack, dim3(S.R), dim3(256), (size_t)(rc_smem(S)), s, D, S, st, full, blk, H);
  return cudaGetLastError();
}
cudaError_t launch_vanilla_commit(const Dims& D, const Sess& S, const DevState& st, const Pass& blk, const Head& H,
                                  cudaStream_t s) {
  static bool a = false;
  if (!a) {
    big_smem(k_vanilla_commit);
    a = true;
  }
  launch_k(k_vanilla_commit, dim3(S.R), dim3(256), (size_t)(rc_smem(S)), s, D, S, st, blk, H);
  return cudaGetLastError();
}

cudaError_t launch_kv_scatter(const Dims& D, const Sess& S, const DevState& st, int r, int k, const float* src,
                              cudaStream_t s) {
  if (D.dtype == 1) launch_k(k_kv_scatter<__nv_bfloat16>, dim3(S.L, D.layers), dim3(256), (size_t)0, s, D, S, st, r, k, src);
  else launch_k(k_kv_scatter<float>, dim3(S.L, D.layers), dim3(256), (size_t)0, s, D, S, st, r, k, src);
  return cudaGetLastError();
}

cudaError_t launch_kv_gather(const Dims& D, const Sess& S, const DevState& st, int r, int k, float* dst,
                             cudaStream_t s) {
  if (D.dtype == 1) launch_k(k_kv_gather<__nv_bfloat16>, dim3(S.L, D.layers), dim3(256), (size_t)0, s, D, S, st, r, k, dst);
  else launch_k(k_kv_gather<float>, dim3(S.L, D.layers), dim3(256), (size_t)0, s, D, S, st, r, k, dst);
  return cudaGetLastError();
}
cudaError_t launch_fresh_pack(const Dims& D, const Sess& S, const DevState& st, const Pass& full, int r, int k,
                              int* save, cudaStream_t s) {
  launch_k(k_fresh_pack, dim3(S.R), dim3(256), (size_t)0, s, D, S, st, full, r, k, save);
  return cudaGetLastError();
}
cudaError_t launch_fresh_restore(const Sess& S, const DevState& st, int r, int k, const int* save, cudaStream_t s) {
  launch_k(k_fresh_restore, dim3(1), dim3(256), (size_t)0, s, S, st, r, k, save);
  return cudaGetLastError();
}
cudaError_t launch_sqdiff_norm(const float* a, const float* b, long long n, double* part, int n_part, double* out,
                               cudaStream_t s) {
  launch_k(k_sqdiff_partial, dim3(n_part), dim3(256), (size_t)0, s, a, b, n, part);
  launch_k(k_sqdiff_final, dim3(1), dim3(32), (size_t)0, s, (const double*)part, n_part, out);
  return cudaGetLastError();
}

}  // namespace bb
