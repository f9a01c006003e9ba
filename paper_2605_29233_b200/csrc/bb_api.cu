// C-ABI implementation: model + session objects, workspace carving, the
// per-iteration kernel sequence (captured once into CUDA graphs) and the
// run_blockbatch loop with asynchronous status polling.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cmath>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: host ranges for nsys / ncu --nvtx

#include "bb200.h"
#include "bb_common.cuh"
#include "bb_gemm.cuh"
#include "bb_layers.cuh"

namespace bb {

struct Model {
  bb_model_desc desc;
  Dims D;
  Weights W;
  float* rope = nullptr;  // owned (cudaMalloc), arch 1
};

struct LayerGemms {
  TcGemm qkv, o, gu, dn;
  SimtGemm sqkv, so, sgu, sdn;
};

struct PassGemms {
  std::vector<LayerGemms> layers;
  int BN = 64;
};

// per-launch GEMM timing (%globaltimer, bb_session_gemm_stats); BB_LIVE_STATS=0
// at session creation leaves it out of the captured kernels
static bool live_stats() {
  const char* e = getenv("BB_LIVE_STATS");
  return !(e && e[0] == '0');
}

struct Session {
  Model* M;
  bb_session_desc desc;
  Dims D;
  Sess S;
  DevState st;
  Pass blk, full;
  Pass fullr;                // stacked refresh: the full pass's buffers, B sequences per request
  bool stack_refresh = false;
  Head H;
  PassGemms gb, gf, gr;
  TcGemm head_tc;
  SimtGemm head_simt;
  float* part = nullptr;
  AttnMaps am{};             // TMA views of the KV pools (bf16 hd-128 attention)
  int* full_rows = nullptr;  // device scalar: rows of the full pass
  int* fullr_rows = nullptr; // device scalar: rows of the stacked refresh pass
  char* ws = nullptr;
  size_t ws_bytes = 0;
  cudaGraphExec_t g_iter = nullptr, g_iter_ref = nullptr, g_prefill = nullptr, g_vanilla = nullptr;
  long long nodes_iter = 0, nodes_iter_ref = 0, nodes_prefill = 0, nodes_vanilla = 0;
  long long kernel_launches = 0, graph_launches = 0;
  unsigned long long* tstat = nullptr;  // [16][8] per-GEMM-kind live timing
  unsigned long long* tsite = nullptr;  // [which 2][kind 5][layer] {min entry, min wait return, max end} (GEMM launch sites)
  bool tsite_on = false;
  unsigned char* ns_tabs = nullptr;     // per-GEMM-shape stream-K piece counts
  size_t ns_used = 0, ns_cap = 0;
  struct NsShape {
    int ntiles, nchunks, KB, G;
    unsigned char* tab;
  };
  std::vector<NsShape> ns_shapes;
  unsigned long long* klog = nullptr;  // BB_KLOG=1: kernel timeline (cudaMalloc'd)
  int* fresh_save = nullptr;           // [n_lp] page-table row saved by bb_fresh_kv
  double* sq_part = nullptr;           // [n_sms] bb_sqdiff_norm partial sums
  int n_sms = 148;                     // queried at session creation
  int tflags = 0;                      // bb_session_desc.test_flags (tests only)
  int32_t* host_ctrl = nullptr;  // pinned [4][R][C_WORDS]
  cudaEvent_t ev[4] = {};
  long long layout[BB_VIEW_COUNT][2];
};

// ------------------------------------------------------------------ helpers
static int fail(int code, const char* msg) {
  if (getenv("BB_DEBUG")) fprintf(stderr, "[bb200] %s\n", msg);
  return code;
}
#define CK(x)                                              \
  do {                                                     \
    cudaError_t e_ = (x);                                  \
    if (e_ != cudaSuccess) {                               \
      if (getenv("BB_DEBUG"))                              \
        fprintf(stderr, "[bb200] %s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return BB_ERR_CUDA;                                  \
    }                                                      \
  } while (0)

struct Carver {
  char* base;
  size_t off = 0;
  bool dry;
  template <typename T>
  T* take(size_t count, size_t align = 256) {
    off = (off + align - 1) / align * align;
    T* p = dry ? nullptr : reinterpret_cast<T*>(base + off);
    off += count * sizeof(T);
    return p;
  }
};

static int round_up(int x, int m) { return (x + m - 1) / m * m; }

static int validate_model(const bb_model_desc* m) {
  if (m->vocab_size < 2 || m->layers < 1 || m->d_model < 1 || m->max_len < 1) return BB_ERR_CONFIG;
  if (m->n_heads < 1 || m->n_kv_heads < 1 || m->n_heads % m->n_kv_heads) return BB_ERR_CONFIG;
  if (m->head_dim != 32 && m->head_dim != 64 && m->head_dim != 128 && m->head_dim != 256) return BB_ERR_CONFIG;
  if (m->dtype != BB_DTYPE_F32 && m->dtype != BB_DTYPE_BF16 && m->dtype != BB_DTYPE_BF16X2) return BB_ERR_CONFIG;
  // split activations ride on the tcgen05 attention (head_dim 128) and the LLaDA-shape layers
  if (m->dtype == BB_DTYPE_BF16X2 && (m->arch != BB_ARCH_LLADA || m->head_dim != 128)) return BB_ERR_CONFIG;
  if (m->arch != BB_ARCH_REF && m->arch != BB_ARCH_LLADA) return BB_ERR_CONFIG;
  if (m->arch == BB_ARCH_REF && (m->n_heads != 1 || m->head_dim != m->d_model || m->d_ff != 0)) return BB_ERR_CONFIG;
  if (m->dtype != BB_DTYPE_F32 && (m->d_model % 64 || (m->d_ff % 64) || (m->n_heads * m->head_dim) % 64))
    return BB_ERR_CONFIG;
  return BB_OK;
}

static Dims make_dims(const bb_model_desc* m) {
  Dims D;
  memset(&D, 0, sizeof(D));
  D.arch = m->arch;
  D.V = m->vocab_size;
  D.n_out = m->vocab_size + 1;
  D.n_ext = m->vocab_size + 2;
  D.layers = m->layers;
  D.d = m->d_model;
  D.nh = m->n_heads;
  D.nkv = m->n_kv_heads;
  D.hd = m->head_dim;
  D.dff = m->d_ff;
  D.max_len = m->max_len;
  D.qkv_bias = m->qkv_bias;
  D.dtype = m->dtype == BB_DTYPE_BF16X2 ? BB_DTYPE_BF16 : m->dtype;  // storage type of weights / activations
  D.split = m->dtype == BB_DTYPE_BF16X2;
  D.qkv_out = (m->n_heads + 2 * m->n_kv_heads) * m->head_dim;
  D.attn_dim = m->n_heads * m->head_dim;
  D.kv_dim = m->n_kv_heads * m->head_dim;
  D.n_vtiles = (D.n_out + 127) / 128;
  D.eps = m->norm_eps;
  D.gamma = m->gamma;
  D.head_scale = m->head_scale;
  D.spike_cut = m->spike_cut;
  D.spike_gain = m->spike_gain;
  D.attn_scale = (float)(1.0 / std::sqrt((double)m->head_dim));
  D.radius = m->radius;
  return D;
}

static size_t esz(const Dims& D) { return D.dtype == BB_DTYPE_BF16 ? 2 : 4; }

// Fixed k-pieces per weight tile for a compacting session's block-pass GEMMs:
// ~2 units per CTA when every row chunk is live (tiles = weight tiles x
// chunks), at least 2 so a batch's tail (one live chunk) still spreads, at
// most 8 (the consumers sum that many planes per element).
static int fixed_np(int tiles, int G, int KB) {
  int np = (2 * G + tiles - 1) / tiles;
  np = np < 2 ? 2 : (np > 8 ? 8 : np);
  return np > KB ? KB : np;
}

// Workspace plan.  dry = size query.
static void plan(Session* s, char* base, bool dry) {
  const Dims& D = s->D;
  Sess& S = s->S;
  Carver c{base, 0, dry};
  const size_t e = esz(D);
  const long long R = S.R, B = S.B, L = S.L;
  DevState& st = s->st;
  auto view = [&](int id, const void* p, size_t bytes) {
    s->layout[id][0] = dry ? 0 : (long long)((const char*)p - base);
    s->layout[id][1] = (long long)bytes;
  };
  st.tokens = c.take<int>(R * B * L);
  view(BB_VIEW_TOKENS, st.tokens, R * B * L * 4);
  st.target = c.take<int>(R * S.G);
  view(BB_VIEW_TARGET, st.target, R * S.G * 4);
  st.prompt = c.take<int>(R * S.P);
  view(BB_VIEW_PROMPT, st.prompt, R * S.P * 4);
  st.init_gen = c.take<int>(R * S.G);
  view(BB_VIEW_INIT_GEN, st.init_gen, R * S.G * 4);
  st.ctrl = c.take<int>(R * C_WORDS);
  view(BB_VIEW_CTRL, st.ctrl, R * C_WORDS * 4);
  st.br = c.take<int>(R * B * B_WORDS);
  view(BB_VIEW_BRANCH, st.br, R * B * B_WORDS * 4);
  st.covered = c.take<uint8_t>(R * B * L);
  view(BB_VIEW_COVERED, st.covered, R * B * L);
  st.pm_h = c.take<char>(R * B * L * D.d * e);
  st.pm_h_lo = D.split ? c.take<char>(R * B * L * D.d * e) : nullptr;
  st.pm_m = c.take<float>(R * B * L);
  view(BB_VIEW_PM_M, st.pm_m, R * B * L * 4);
  st.pm_s = c.take<float>(R * B * L);
  view(BB_VIEW_PM_S, st.pm_s, R * B * L * 4);
  st.pm_boost = c.take<float>(R * B * L);
  st.pt = c.take<int>(R * B * S.n_lp);
  view(BB_VIEW_PAGES, st.pt, R * B * S.n_lp * 4);
  st.refc = c.take<int>(R * S.pool);
  view(BB_VIEW_REFC, st.refc, R * S.pool * 4);
  st.freel = c.take<int>(R * S.pool);
  st.free_top = c.take<int>(R);
  st.copies = c.take<int>(R * S.max_copies * 2);
  st.pm_copies = c.take<int>(R * MAXB * 2);
  st.events = c.take<int>(R * (long long)S.ev_cap * EVW);
  view(BB_VIEW_EVENTS, st.events, R * (long long)S.ev_cap * EVW * 4);
  st.ptab = c.take<float>(R * B * L * B);
  st.ptab_ok = c.take<uint8_t>(R * B * L);
  const long long kv_el = (long long)D.layers * R * S.pool * D.nkv * S.ps * D.hd;
  // split: each pool is followed by its lo pool (same layout, kv_lo elements on)
  st.kv_lo = D.split ? kv_el : 0;
  st.kv_k = c.take<char>(kv_el * e * (D.split ? 2 : 1), 1024);
  st.kv_v = c.take<char>(kv_el * e * (D.split ? 2 : 1), 1024);

  auto pass = [&](Pass& P, int rows_alloc, int max_items, int item_rows, int full, int groups) {
    P.rows_alloc = rows_alloc;
    P.full = full;
    P.item_rows = item_rows;
    P.slot_pos = c.take<int>(rows_alloc);
    P.slot_req = c.take<int>(rows_alloc);
    P.slot_br = c.take<int>(rows_alloc);
    P.slot_tok = c.take<int>(rows_alloc);
    P.slot_kvoff = c.take<long long>(rows_alloc);
    P.rng_off = c.take<int>(R * MAXB);
    P.rng_cnt = c.take<int>(R * MAXB);
    P.items = c.take<int>(R * max_items * ITW);
    P.n_items = c.take<int>(R);
    P.skip = c.take<int>(1);
    P.x = c.take<float>((long long)rows_alloc * D.d);
    P.xn = c.take<char>((long long)rows_alloc * D.d * e, 1024);
    P.q = c.take<char>((long long)rows_alloc * D.attn_dim * e, 1024);
    P.attn = c.take<char>((long long)rows_alloc * D.attn_dim * e, 1024);
    P.act = c.take<char>((long long)rows_alloc * (D.dff > 0 ? D.dff : 1) * e, 1024);
    P.xn_lo = P.q_lo = P.attn_lo = P.act_lo = nullptr;
    if (D.split) {
      P.xn_lo = c.take<char>((long long)rows_alloc * D.d * e, 1024);
      P.q_lo = c.take<char>((long long)rows_alloc * D.attn_dim * e, 1024);
      P.attn_lo = c.take<char>((long long)rows_alloc * D.attn_dim * e, 1024);
      P.act_lo = c.take<char>((long long)rows_alloc * (D.dff > 0 ? D.dff : 1) * e, 1024);
    }
    P.apart = c.take<float>(R * max_items * (long long)item_rows * D.nh * (D.hd + 2));
    P.row_rope = (!full && D.arch == BB_ARCH_LLADA) ? c.take<float>((long long)rows_alloc * D.hd) : nullptr;
    // the M = 128 tcgen05 attention (bf16, hd 128, 16-row pages) reads 128-row key tiles: block
    // passes with > 64 rows per request (C5 windows: 120) and long full passes (L >= 1024; C5
    // 484 vs 633 us per launch); short full passes and <= 64-row windows keep the 64-row kernel
    // (two CTAs per SM, no half-empty tiles; C2 full pass 14.9 vs 26.3 us)
#ifndef ATT_F8_MIN_ROWS
#define ATT_F8_MIN_ROWS 64  // block passes with more rows per request use the 128-row attention
#endif
    P.kz_shift = (D.dtype == BB_DTYPE_BF16 && D.hd == 128 && S.ps == 16 && !(s->tflags & 7) &&
                  (full ? S.L >= 1024 : item_rows > ATT_F8_MIN_ROWS)) ? 7 : 6;
    P.n_kz = full ? 1 : (item_rows + (1 << P.kz_shift) - 1) >> P.kz_shift;
    P.akey_cap = B * S.n_lp * S.ps;  // every page segment padded to ps entries
    P.akeys = c.take<int>((long long)groups * P.n_kz * P.akey_cap * 2);
    P.akey_n = c.take<int>((long long)groups * P.n_kz * 2);
    P.req_base = c.take<int>(R);
    P.rows_live = c.take<int>(1);
  };
  pass(s->blk, round_up(S.NR, s->gb.BN), S.max_items, S.NRq, 0, S.R);
  {
    // the stacked refresh pass shares the full pass's buffers (sized for the larger)
    const int rows_f = round_up(S.NF, s->gf.BN);
    const int rows_r = s->stack_refresh ? round_up(S.NF * S.B, s->gr.BN) : 0;
    pass(s->full, rows_f > rows_r ? rows_f : rows_r, 1, S.L, 1, s->stack_refresh ? S.R * S.B : S.R);
    s->full.rows_alloc = rows_f;
    s->fullr = s->full;
    s->fullr.rows_alloc = rows_r;
    s->fullr.nseq = S.B;
  }
  Head& H = s->H;
  const int rb = s->blk.rows_alloc;
  H.masked = c.take<int>(rb);
  H.boost = c.take<float>(rb);
  H.tgt = c.take<int>(rb);
  H.hpart = c.take<float4>((long long)rb * D.n_vtiles);
  H.logits = D.dtype == BB_DTYPE_F32 ? c.take<float>((long long)rb * D.n_out) : nullptr;
  H.raw = (D.dtype == BB_DTYPE_BF16 && (s->desc.logits || s->desc.seam)) ? c.take<float>((long long)rb * D.n_out) : nullptr;
  H.res_conf = c.take<float>(rb);
  H.res_arg = c.take<int>(rb);
  H.res_m = c.take<float>(rb);
  H.res_s = c.take<float>(rb);
  view(BB_VIEW_HEAD_MASKED, H.masked, (size_t)rb * 4);
  view(BB_VIEW_HEAD_M, H.res_m, (size_t)rb * 4);
  view(BB_VIEW_HEAD_S, H.res_s, (size_t)rb * 4);
  view(BB_VIEW_HEAD_ARG, H.res_arg, (size_t)rb * 4);
  view(BB_VIEW_SLOT_POS, s->blk.slot_pos, (size_t)rb * 4);
  view(BB_VIEW_SLOT_BR, s->blk.slot_br, (size_t)rb * 4);
  H.skip = c.take<int>(1);
  s->full_rows = c.take<int>(1);
  s->fullr_rows = c.take<int>(1);
  s->tstat = c.take<unsigned long long>(17 * 8);  // slot 16: GEMM phase marks (BB_GEMM_PH builds)
  s->tsite = c.take<unsigned long long>((size_t)3 * 10 * D.layers);
  s->tsite_on = live_stats();
  s->blk.atstat = s->tstat + 5 * 8;   // slots 5/6: block-pass attention (duration, start spread)
  s->full.atstat = s->tstat + 13 * 8; // slots 13/14: full-pass attention
  s->fullr.atstat = s->full.atstat;
  s->fresh_save = c.take<int>(S.n_lp);
  s->sq_part = c.take<double>(1024);
  s->ns_cap = 64 * 1024;
  s->ns_tabs = c.take<unsigned char>(s->ns_cap);
  // GEMM partial planes: max over all stream-K GEMMs of (slots x rows x n_out)
  long long part = 1;
  if (D.dtype == BB_DTYPE_BF16) {
    const int outs[4] = {D.qkv_out, D.d, 2 * D.dff, D.d};
    const int ks[4] = {D.d, D.attn_dim, D.d, D.dff};
    for (int which = 0; which < (s->stack_refresh ? 3 : 2); ++which) {
      const int rows = which == 0 ? s->blk.rows_alloc : (which == 1 ? s->full.rows_alloc : s->fullr.rows_alloc);
      const int BN = which == 0 ? s->gb.BN : (which == 1 ? s->gf.BN : s->gr.BN);
      for (int g = 0; g < 4; ++g) {
        if (outs[g] == 0) continue;
        const int ntiles = (outs[g] + 127) / 128, nch_all = rows / BN, KB = (ks[g] + 63) / 64;
        const long long T_all = (long long)ntiles * nch_all * KB;
        const int G = (int)(T_all < s->n_sms ? T_all : s->n_sms);
        int ms = 1;
        if (which == 0 && S.compact) {
          ms = fixed_np(ntiles * nch_all, G, KB);  // fixed pieces per tile
        } else {
          for (long long t = 0; t < (long long)ntiles * nch_all; ++t) {
            const int ns = sk_owner(t * KB + KB - 1, T_all, G) - sk_owner(t * KB, T_all, G) + 1;
            ms = ns > ms ? ns : ms;
          }
        }
        const long long need = (long long)ms * rows * outs[g];
        part = need > part ? need : part;
      }
    }
  } else {
    // SIMT GEMMs write every allocated row of their pass (block passes can
    // have more rows than the full pass: a seam session's 192-row full pass
    // vs its 256-row block pass)
    const int outs[4] = {D.qkv_out, D.d, 2 * D.dff, D.d};
    const long long rows = std::max(s->blk.rows_alloc, s->full.rows_alloc);
    for (int g = 0; g < 4; ++g) {
      const long long need = rows * outs[g];
      part = need > part ? need : part;
    }
  }
  s->part = c.take<float>(part);
  s->ws_bytes = c.off + 1024;
}

static PartRef pref_tc(const TcGemm& g, const float* part) {
  return PartRef{part, g.p.plane, g.p.ldp, g.sk};
}

// per-tile stream-K piece counts (avoids 64-bit divisions in consumers);
// one table per distinct GEMM shape (all layers share them)
#ifndef GEMM_RR_ROUNDS
#define GEMM_RR_ROUNDS 12  // full-pass GEMMs with at least this many rounds of whole tiles run mode 2
#endif
static int attach_ns_table(Session* s, TcGemm& g) {
  const long long tiles = (long long)g.p.n_ntiles * g.p.n_chunks;
  for (auto& e : s->ns_shapes)
    if (e.ntiles == g.p.n_ntiles && e.nchunks == g.p.n_chunks && e.KB == g.sk.KB && e.G == g.sk.G) {
      g.sk.ns_tab = e.tab;
      return BB_OK;
    }
  if (s->ns_used + tiles > s->ns_cap) return BB_ERR_NOMEM;
  std::vector<unsigned char> tab(tiles);
  for (long long t = 0; t < tiles; ++t)
    tab[t] = (unsigned char)(sk_owner(t * g.sk.KB + g.sk.KB - 1, g.sk.T, g.sk.G) - sk_owner(t * g.sk.KB, g.sk.T, g.sk.G) + 1);
  unsigned char* dst = s->ns_tabs + s->ns_used;
  if (cudaMemcpy(dst, tab.data(), tiles, cudaMemcpyHostToDevice) != cudaSuccess) return BB_ERR_CUDA;
  g.sk.ns_tab = dst;
  s->ns_used += (tiles + 15) / 16 * 16;
  s->ns_shapes.push_back({g.p.n_ntiles, g.p.n_chunks, g.sk.KB, g.sk.G, dst});
  return BB_OK;
}

static int setup_gemms(Session* s) {
  const Dims& D = s->D;
  const Weights& W = s->M->W;
  const size_t e = esz(D);
  // block pass: the attention CTAs prefetch the O projection's weights into
  // L2 while they run (HBM is otherwise idle during the attention)
  s->blk.pf_base = nullptr;
  s->full.pf_base = nullptr;
  if (D.dtype == BB_DTYPE_BF16) {
    s->blk.pf_base = (const char*)W.wo;
    s->blk.pf_layer_bytes = (long long)D.d * D.attn_dim * (long long)e;
  }
  s->fullr.pf_base = nullptr;
  for (int which = 0; which < (s->stack_refresh ? 3 : 2); ++which) {
    Pass& P = which == 0 ? s->blk : (which == 1 ? s->full : s->fullr);
    PassGemms& G = which == 0 ? s->gb : (which == 1 ? s->gf : s->gr);
    int* rows_full = which == 2 ? s->fullr_rows : s->full_rows;
    G.layers.resize(D.layers);
    for (int l = 0; l < D.layers; ++l) {
      LayerGemms& lg = G.layers[l];
      const char* wqkv = (const char*)W.wqkv + (size_t)l * D.qkv_out * D.d * e;
      const char* wo = (const char*)W.wo + (size_t)l * D.d * D.attn_dim * e;
      const char* wgu = D.dff ? (const char*)W.wgu + (size_t)l * 2 * D.dff * D.d * e : nullptr;
      const char* wd = D.dff ? (const char*)W.wd + (size_t)l * D.d * D.dff * e : nullptr;
      if (D.dtype == BB_DTYPE_BF16) {
        if (!tc_gemm_setup(lg.qkv, wqkv, D.qkv_out, D.d, P.xn, P.rows_alloc, G.BN, 0, s->n_sms, P.xn_lo))
          return BB_ERR_CONFIG;
        if (!tc_gemm_setup(lg.o, wo, D.d, D.attn_dim, P.attn, P.rows_alloc, G.BN, 0, s->n_sms, P.attn_lo))
          return BB_ERR_CONFIG;
        if (D.dff) {
          if (!tc_gemm_setup(lg.gu, wgu, 2 * D.dff, D.d, P.xn, P.rows_alloc, G.BN, 0, s->n_sms, P.xn_lo))
            return BB_ERR_CONFIG;
          if (!tc_gemm_setup(lg.dn, wd, D.d, D.dff, P.act, P.rows_alloc, G.BN, 0, s->n_sms, P.act_lo))
            return BB_ERR_CONFIG;
        }
        TcGemm* all[4] = {&lg.qkv, &lg.o, &lg.gu, &lg.dn};
        for (int g = 0; g < (D.dff ? 4 : 2); ++g) {
          GemmTcParams& p = all[g]->p;
          const int wk = which > 1 ? 1 : which;  // the stacked refresh reports as a full pass
          p.tstat = s->tsite_on ? s->tsite + 3 * ((size_t)(wk * 5 + g) * D.layers + l) : nullptr;
          p.klog = s->D.klog;
          p.klog_cap = s->D.klog_cap;
          p.klog_id = 100 + wk * 8 + g;
          if (which >= 1 && !(s->tflags & 1024)) {
            // large full passes: whole tiles in L2-friendly groups (test flag 1024: stream-K)
            const int kin = g == 1 ? D.attn_dim : (g == 3 ? D.dff : D.d);
            tc_gemm_round_robin(*all[g], GEMM_RR_ROUNDS, kin * 2 * (P.xn_lo != nullptr ? 2 : 1));
          }
          if (p.mode == 0 && attach_ns_table(s, *all[g]) != BB_OK) return BB_ERR_NOMEM;
          p.part = s->part;
          p.skip = P.skip;
          p.rows_valid = which >= 1 ? rows_full : nullptr;
          if (which == 0 && s->S.compact) {
            // batched: fixed k-pieces per tile (sums independent of how many requests are
            // live) and only the live requests' row chunks (test flag 256: all chunks)
            p.np = all[g]->sk.np = fixed_np(p.n_ntiles * p.n_chunks, all[g]->grid, p.KB);
            if (!(s->tflags & 256)) p.rows_valid = p.rows_dyn = s->blk.rows_live;
          }
        }
      } else {
        lg.sqkv = SimtGemm{(const float*)wqkv, (const float*)P.xn, D.qkv_out, D.d, P.rows_alloc,
                           which >= 1 ? rows_full : nullptr, P.skip, s->part, D.qkv_out};
        lg.so = SimtGemm{(const float*)wo, (const float*)P.attn, D.d, D.attn_dim, P.rows_alloc,
                         which >= 1 ? rows_full : nullptr, P.skip, s->part, D.d};
        if (D.dff) {
          lg.sgu = SimtGemm{(const float*)wgu, (const float*)P.xn, 2 * D.dff, D.d, P.rows_alloc,
                            which >= 1 ? rows_full : nullptr, P.skip, s->part, 2 * D.dff};
          lg.sdn = SimtGemm{(const float*)wd, (const float*)P.act, D.d, D.dff, P.rows_alloc,
                            which >= 1 ? rows_full : nullptr, P.skip, s->part, D.d};
        }
      }
    }
  }
  s->am.ok = false;
  if (D.dtype == BB_DTYPE_BF16 && D.hd == 128 && s->S.ps == 16) {
    attn_prepare();
    const uint64_t rows = (uint64_t)D.layers * s->S.R * s->S.pool * D.nkv * s->S.ps;
    s->am.ok = tma_map_bf16(&s->am.k, s->st.kv_k, (uint64_t)D.hd, rows, 16) &&
               tma_map_bf16(&s->am.v, s->st.kv_v, (uint64_t)D.hd, rows, 16);
    s->am.kl = s->am.k;
    s->am.vl = s->am.v;
    if (s->am.ok && D.split)
      s->am.ok = tma_map_bf16(&s->am.kl, (const __nv_bfloat16*)s->st.kv_k + s->st.kv_lo, (uint64_t)D.hd, rows, 16) &&
                 tma_map_bf16(&s->am.vl, (const __nv_bfloat16*)s->st.kv_v + s->st.kv_lo, (uint64_t)D.hd, rows, 16);
  }
  if (D.dtype == BB_DTYPE_BF16) {
    if (!tc_gemm_setup(s->head_tc, W.head, D.n_out, D.d, s->blk.xn, s->blk.rows_alloc, s->gb.BN, 1, s->n_sms,
                       s->blk.xn_lo))
      return BB_ERR_CONFIG;
    GemmTcParams& p = s->head_tc.p;
    p.head_part = s->H.hpart;
    p.raw_out = s->H.raw;
    p.boost = s->H.boost;
    p.tgt = s->H.tgt;
    p.head_scale = D.head_scale;
    p.spike_cut = D.spike_cut;
    p.spike_gain = D.spike_gain;
    p.skip = s->H.skip;
    if (s->S.compact && !(s->tflags & (256 | 512))) p.rows_valid = p.rows_dyn = s->blk.rows_live;
    p.tstat = s->tsite_on ? s->tsite + 3 * ((size_t)4 * D.layers) : nullptr;
    p.klog = s->D.klog;
    p.klog_cap = s->D.klog_cap;
    p.klog_id = 104;
  } else {
    s->head_simt = SimtGemm{(const float*)W.head, (const float*)s->blk.xn, D.n_out, D.d, s->blk.rows_alloc,
                            nullptr, s->H.skip, s->H.logits, D.n_out};
  }
  return BB_OK;
}

static PartRef pref_simt(const SimtGemm& g) {
  SplitK sk{};
  return PartRef{g.out, 0, g.ldo, sk};
}

// ------------------------------------------------------------------ forward pass
// GEMM launch sites -> per kind (block 0-3, full 8-11, head 4) in tstat[kind]:
// [3] += max end - min kernel entry (the launch's whole duration, its pre-wait
// weight prefetch included), [2] += max end - min dependency-wait return,
// [4] += 1; sites reset for the next pass
__global__ void k_tsite_fold(unsigned long long* site, int n_layers, unsigned long long* tstat) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 10 * n_layers) return;
  unsigned long long* t = site + 3 * (size_t)i;
  const unsigned long long t0 = t[0], tw = t[1], t1 = t[2];
  if (t0 == ~0ull || t1 == 0ull) return;
  const int sk = i / n_layers, which = sk / 5, kind = sk % 5;
  unsigned long long* dst = tstat + 8 * (kind == 4 ? 4 : which * 8 + kind);
  atomicAdd(&dst[3], t1 > t0 ? t1 - t0 : 0ull);
  atomicAdd(&dst[2], (tw != ~0ull && t1 > tw) ? t1 - tw : 0ull);
  atomicAdd(&dst[4], 1ull);
  t[0] = ~0ull;
  t[1] = ~0ull;
  t[2] = 0ull;
}

static cudaError_t tsite_fold(Session* s, cudaStream_t st) {
  if (!s->tsite_on) return cudaSuccess;
  const int n = 10 * s->D.layers;
  k_tsite_fold<<<(n + 127) / 128, 128, 0, st>>>(s->tsite, s->D.layers, s->tstat);
  return cudaGetLastError();
}

static cudaError_t run_gemm(Session* s, const TcGemm& tg, const SimtGemm& sg, PartRef* pr, cudaStream_t st) {
  if (s->D.dtype == BB_DTYPE_BF16) {
    *pr = pref_tc(tg, s->part);
    return tc_gemm_launch(tg, st);
  }
  *pr = pref_simt(sg);
  return simt_gemm_launch(sg, st);
}

static cudaError_t forward(Session* s, Pass& P, PassGemms& G, cudaStream_t st) {
  const Dims& D = s->D;
  const Weights& W = s->M->W;
  cudaError_t e;
  if ((e = launch_embed(D, s->S, P, W, st)) != cudaSuccess) return e;
  for (int l = 0; l < D.layers; ++l) {
    LayerGemms& lg = G.layers[l];
    const float* next_ln = l + 1 < D.layers ? (D.arch == BB_ARCH_LLADA ? W.ln1 + (size_t)(l + 1) * D.d : nullptr)
                                            : (D.arch == BB_ARCH_LLADA ? W.lnf : nullptr);
    PartRef pr;
    if ((e = run_gemm(s, lg.qkv, lg.sqkv, &pr, st)) != cudaSuccess) return e;
    if ((e = launch_post_qkv(D, s->S, P, s->st, W, l, pr, st)) != cudaSuccess) return e;
    if ((e = launch_attn(D, s->S, P, s->st, s->am, l, s->tflags, st)) != cudaSuccess) return e;
    if ((e = run_gemm(s, lg.o, lg.so, &pr, st)) != cudaSuccess) return e;
    if (D.dff) {
      if ((e = launch_post_residual(D, P, pr, W.ln2 + (size_t)l * D.d, st)) != cudaSuccess) return e;
      if ((e = run_gemm(s, lg.gu, lg.sgu, &pr, st)) != cudaSuccess) return e;
      if ((e = launch_post_gu(D, P, pr, st)) != cudaSuccess) return e;
      if ((e = run_gemm(s, lg.dn, lg.sdn, &pr, st)) != cudaSuccess) return e;
      if ((e = launch_post_residual(D, P, pr, next_ln, st)) != cudaSuccess) return e;
    } else {
      if ((e = launch_post_residual(D, P, pr, next_ln, st)) != cudaSuccess) return e;
    }
  }
  return tsite_fold(s, st);
}

static cudaError_t head(Session* s, cudaStream_t st) {
  const Dims& D = s->D;
  cudaError_t e;
  if (D.dtype == BB_DTYPE_BF16) {
    if ((e = tc_gemm_launch(s->head_tc, st)) != cudaSuccess) return e;
    if ((e = tsite_fold(s, st)) != cudaSuccess) return e;
  } else {
    if ((e = simt_gemm_launch(s->head_simt, st)) != cudaSuccess) return e;
    if ((e = launch_head_tiles_f32(D, s->blk, s->H, st)) != cudaSuccess) return e;
  }
  return launch_head_reduce(D, s->S, s->blk, s->H, s->st, st);
}

// prefill in two parts (the diagnostics mode reads the caches in between):
// 0 = init + full forward + head, 1 = first commits, merge/sync, copies
static int enqueue_prefill_part(Session* s, int part, cudaStream_t st) {
  const Dims& D = s->D;
  const Sess& S = s->S;
  if (part == 0) {
    CK(launch_prefill_init(D, S, s->st, s->full, s->blk, s->H, st));
    CK(launch_attn_keys(D, S, s->full, s->st, st));
    CK(forward(s, s->full, s->gf, st));
    CK(launch_gather_head(D, S, s->full, s->blk, s->H, -1, st));
    CK(head(s, st));
  } else {
    CK(launch_prefill_post(D, S, s->st, s->blk, s->H, st));
    CK(launch_merge_prep(D, S, s->st, s->M->W, st));
    CK(launch_merge_sync(D, S, s->st, 1, st));
    CK(launch_copy_pages(D, S, s->st, 1, st));
  }
  return BB_OK;
}

static int enqueue_prefill(Session* s, cudaStream_t st) {
  const int rc = enqueue_prefill_part(s, 0, st);
  return rc != BB_OK ? rc : enqueue_prefill_part(s, 1, st);
}

// block step in three parts: 0 = pack + copy-on-write copies (ctrl then holds
// the active set), 1 = forward + head, 2 = commit, EOS, merge/sync, copies
static int enqueue_block_step_part(Session* s, int part, cudaStream_t st) {
  const Dims& D = s->D;
  const Sess& S = s->S;
  if (part == 0) {
    CK(cudaMemsetAsync(s->blk.skip, 1, sizeof(int), st));
    CK(cudaMemsetAsync(s->H.skip, 1, sizeof(int), st));
    if (S.compact) CK(launch_block_bases(D, S, s->st, s->blk, s->H, st));
    CK(launch_block_pack(D, S, s->st, s->blk, s->H, st));
    CK(launch_copy_pages(D, S, s->st, 0, st));
  } else if (part == 1) {
    CK(launch_attn_keys(D, S, s->blk, s->st, st));
    CK(forward(s, s->blk, s->gb, st));
    CK(head(s, st));
  } else {
    CK(launch_step_commit(D, S, s->st, s->blk, s->H, st));
    CK(launch_merge_prep(D, S, s->st, s->M->W, st));
    CK(launch_merge_sync(D, S, s->st, 0, st));
    CK(launch_copy_pages(D, S, s->st, 1, st));
  }
  return BB_OK;
}

static int enqueue_block_step(Session* s, cudaStream_t st) {
  for (int part = 0; part < 3; ++part) {
    const int rc = enqueue_block_step_part(s, part, st);
    if (rc != BB_OK) return rc;
  }
  return BB_OK;
}

static int enqueue_refresh(Session* s, cudaStream_t st) {
  const Dims& D = s->D;
  const Sess& S = s->S;
  CK(cudaMemsetAsync(s->H.skip, 1, sizeof(int), st));
  if (s->stack_refresh) {
    // every refreshing branch in one B x L pass: the weights stream once per
    // refresh instead of once per branch (refresh loop, scheduler.py:379-383)
    CK(cudaMemsetAsync(s->fullr.skip, 1, sizeof(int), st));
    CK(launch_refresh_pack(D, S, s->st, s->fullr, s->blk, s->H, -1, st));
    CK(launch_attn_keys(D, S, s->fullr, s->st, st));
    CK(forward(s, s->fullr, s->gr, st));
    CK(launch_gather_head(D, S, s->fullr, s->blk, s->H, -1, st));
    // rows [R*L, R*B*L) are padding of the R*L-row passes (prefill, vanilla,
    // fresh_kv): back to -1, or their post kernels would write the stale rows'
    // K/V into the next request's pages
    CK(cudaMemsetAsync(s->full.slot_pos + S.NF, 0xFF, (size_t)(s->fullr.rows_alloc - S.NF) * sizeof(int), st));
    CK(head(s, st));
    CK(launch_refresh_end(D, S, s->st, st));
    return BB_OK;
  }
  for (int k = 0; k < S.B; ++k) {
    CK(cudaMemsetAsync(s->full.skip, 1, sizeof(int), st));
    CK(launch_refresh_pack(D, S, s->st, s->full, s->blk, s->H, k, st));
    CK(launch_attn_keys(D, S, s->full, s->st, st));
    CK(forward(s, s->full, s->gf, st));
    CK(launch_gather_head(D, S, s->full, s->blk, s->H, k, st));
  }
  CK(head(s, st));
  CK(launch_refresh_end(D, S, s->st, st));
  return BB_OK;
}

// one vanilla_decode round (decoding.py:279-321): full forward of branch 0,
// head over the masked positions before the first eos, Eq. 1 with tau 1.0
static int enqueue_vanilla(Session* s, cudaStream_t st) {
  const Dims& D = s->D;
  const Sess& S = s->S;
  CK(cudaMemsetAsync(s->full.skip, 1, sizeof(int), st));
  CK(cudaMemsetAsync(s->H.skip, 1, sizeof(int), st));
  CK(launch_vanilla_pack(D, S, s->st, s->full, s->blk, s->H, st));
  CK(launch_attn_keys(D, S, s->full, s->st, st));
  CK(forward(s, s->full, s->gf, st));
  CK(launch_gather_head(D, S, s->full, s->blk, s->H, 0, st));
  CK(head(s, st));
  CK(launch_vanilla_commit(D, S, s->st, s->blk, s->H, st));
  return BB_OK;
}

static long long count_kernel_nodes(cudaGraph_t g) {
  size_t n = 0;
  if (cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess) return -1;
  std::vector<cudaGraphNode_t> nodes(n);
  cudaGraphGetNodes(g, nodes.data(), &n);
  long long k = 0;
  for (size_t i = 0; i < n; ++i) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nodes[i], &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}

// what: 0 = block step, 1 = block step + refresh, 2 = prefill, 3 = vanilla round
static int capture(Session* s, int what, cudaStream_t st, cudaGraphExec_t* out, long long* nodes) {
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  int rc = what == 2 ? enqueue_prefill(s, st) : (what == 3 ? enqueue_vanilla(s, st) : enqueue_block_step(s, st));
  if (rc == BB_OK && what == 1) rc = enqueue_refresh(s, st);
  cudaError_t e = cudaStreamEndCapture(st, &g);
  if (rc != BB_OK) return rc;
  CK(e);
  *nodes = count_kernel_nodes(g);
  CK(cudaGraphInstantiate(out, g, 0));
  cudaGraphDestroy(g);
  return BB_OK;
}

}  // namespace bb

using namespace bb;

extern "C" {

BB_API int bb_version(void) { return 1; }

BB_API int bb_model_create(const bb_model_desc* desc, const bb_weights* w, void** out) {
  if (!desc || !w || !out) return BB_ERR_CONTRACT;
  int rc = validate_model(desc);
  if (rc != BB_OK) return fail(rc, "invalid model desc");
  Model* m = new Model();
  m->desc = *desc;
  m->D = make_dims(desc);
  m->W.emb = w->emb;
  m->W.pos = w->pos;
  m->W.wqkv = w->wqkv;
  m->W.bqkv = desc->qkv_bias ? w->bqkv : nullptr;
  m->W.wo = w->wo;
  m->W.wgu = w->wgu;
  m->W.wd = w->wd;
  m->W.ln1 = w->ln1;
  m->W.ln2 = w->ln2;
  m->W.lnf = w->lnf;
  m->W.head = w->head;
  if (desc->arch == BB_ARCH_LLADA) {
    const int half = desc->head_dim / 2;
    std::vector<float> tab((size_t)desc->max_len * half * 2);
    for (int p = 0; p < desc->max_len; ++p)
      for (int i = 0; i < half; ++i) {
        const double inv = std::pow((double)desc->rope_theta, -2.0 * i / desc->head_dim);
        const double a = (double)p * inv;
        tab[((size_t)p * half + i) * 2] = (float)std::cos(a);
        tab[((size_t)p * half + i) * 2 + 1] = (float)std::sin(a);
      }
    if (cudaMalloc(&m->rope, tab.size() * 4) != cudaSuccess) {
      delete m;
      return BB_ERR_CUDA;
    }
    cudaMemcpy(m->rope, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice);
  }
  m->W.rope = m->rope;
  *out = m;
  return BB_OK;
}

BB_API int bb_model_destroy(void* model) {
  Model* m = (Model*)model;
  if (!m) return BB_OK;
  if (m->rope) cudaFree(m->rope);
  delete m;
  return BB_OK;
}

static int make_session(Model* M, const bb_session_desc* d, Session* s) {
  s->M = M;
  s->desc = *d;
  s->D = M->D;
  {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
        sms > 0)
      s->n_sms = sms > 1024 ? 1024 : sms;
    s->tflags = d->test_flags;
  }
  Sess& S = s->S;
  memset(&S, 0, sizeof(S));
  if (d->n_requests < 1 || d->n_branches < 1 || d->n_branches > MAXB) return BB_ERR_CONFIG;
  if (d->prompt_len < 1 || d->gen_len < 1) return BB_ERR_CONFIG;
  if (!(d->tau_conf >= 0.f && d->tau_conf <= 1.f) || !(d->tau_merge >= 0.f && d->tau_merge <= 1.f)) return BB_ERR_CONFIG;
  if (d->tau_sync < 0 || d->refresh_interval < 1) return BB_ERR_CONFIG;
  S.R = d->n_requests;
  S.B = d->n_branches;
  S.P = d->prompt_len;
  S.G = d->gen_len;
  S.L = S.P + S.G;
  if (S.L > M->D.max_len) return BB_ERR_CONTRACT;  // model.py:286-287
  int off = 0, maxb = 0;
  for (int k = 0; k < S.B; ++k) {
    if (d->block_sizes[k] < 1) return BB_ERR_CONFIG;
    for (int j = 0; j < k; ++j)
      if (d->block_sizes[j] == d->block_sizes[k]) return BB_ERR_CONFIG;
    S.bs[k] = d->block_sizes[k];
    S.off[k] = off;
    off += S.bs[k];
    maxb = maxb > S.bs[k] ? maxb : S.bs[k];
  }
  S.NRq = off;
  S.NR = S.R * S.NRq;
  S.NF = S.R * S.L;
  S.tau_conf = d->tau_conf;
  S.tau_merge = d->tau_merge;
  S.tau_sync = d->tau_sync;
  S.refresh_interval = d->refresh_interval;
  S.merge_en = d->merge_enabled;
  S.sync_en = d->sync_enabled;
  S.ps = d->page_size > 0 ? d->page_size : 16;
  if (S.ps > 32 || (S.ps & (S.ps - 1)) != 0) return BB_ERR_CONFIG;  // power of two <= 32
  S.ps_shift = 0;
  while ((1 << S.ps_shift) < S.ps) ++S.ps_shift;
  S.n_pp = (S.P + S.ps - 1) / S.ps;
  S.n_gp = (S.G + S.ps - 1) / S.ps;
  S.n_lp = S.n_pp + S.n_gp;
  S.diag = d->diagnostics ? 1 : 0;
  S.n_sms = s->n_sms;
  S.pool = S.B * S.n_lp + (S.diag ? S.n_lp : 0);
  S.ch_block = d->pages_per_item > 0 ? d->pages_per_item : 4;
  S.max_items = S.B * ((S.n_lp + S.ch_block - 1) / S.ch_block) + 2 * S.B + 4;
  S.ev_cap = d->event_capacity > 0 ? d->event_capacity : 32768;
  S.trace = d->trace;
  S.hard_cap = d->hard_cap > 0 ? d->hard_cap : 4 * S.G * S.B + 16;  // scheduler.py:310
  S.max_copies = S.B * (maxb / S.ps + 2);
  // test flag bit 3: keep the static block-pass layout in a batched session (A/B)
  S.compact = (S.R > 1 && s->D.dtype == BB_DTYPE_BF16 && !d->seam && !d->diagnostics && !(d->test_flags & 8)) ? 1 : 0;
  const int NR = S.NR;
  // rows per GEMM chunk (bf16x2: the MMA's N holds each row twice, hi and lo,
  // so chunks carry at most 128 rows)
  const bool split = s->D.split != 0;
  s->gb.BN = NR <= 64 ? 64 : ((NR <= 128 || split) ? 128 : 256);
  // full pass (prefill / refresh): row chunks as wide as possible with little
  // padding (L = 320 -> 2 x 160, L = 192 -> 1 x 192, L = 3072 -> 12 x 256)
  auto full_bn = [&](long long rows) {
    // (the epilogue reads 32 accumulator columns at a time: rows per chunk % 32 == 0)
    const int cands_n[5] = {256, 192, 160, 128, 64}, cands_s[3] = {128, 96, 64};
    const int* cands = split ? cands_s : cands_n;
    const int n_c = split ? 3 : 5;
    int best = 128;
    long long best_cost = -1;
    for (int i = 0; i < n_c; ++i) {
      const int bn = cands[i];
      const long long chunks = (rows + bn - 1) / bn;
      const long long cost = chunks * bn + chunks * 32;  // padded rows + per-chunk weight re-read penalty
      if (best_cost < 0 || cost < best_cost) {
        best_cost = cost;
        best = bn;
      }
    }
    return best;
  };
  s->gf.BN = full_bn(S.NF);
  // refresh: every refreshing branch stacked into one B x L pass on the
  // key-list attention paths (the per-branch SIMT items keep one pass per
  // branch; test flag bit 11 forces that everywhere)
  s->stack_refresh = s->D.dtype == BB_DTYPE_BF16 && !uses_items(s->D) && S.B > 1 && !(d->test_flags & 2048);
  s->gr.BN = s->stack_refresh ? full_bn((long long)S.NF * S.B) : s->gf.BN;
  return BB_OK;
}

BB_API int bb_session_workspace_bytes(const void* model, const bb_session_desc* d, size_t* bytes) {
  if (!model || !d || !bytes) return BB_ERR_CONTRACT;
  Session s;
  int rc = make_session((Model*)model, d, &s);
  if (rc != BB_OK) return rc;
  plan(&s, nullptr, true);
  *bytes = s.ws_bytes;
  return BB_OK;
}

BB_API int bb_session_create(void* model, const bb_session_desc* d, void* workspace, size_t bytes, void** out) {
  if (!model || !d || !workspace || !out) return BB_ERR_CONTRACT;
  Session* s = new Session();
  int rc = make_session((Model*)model, d, s);
  if (rc != BB_OK) {
    delete s;
    return rc;
  }
  char* base = (char*)(((uintptr_t)workspace + 1023) & ~(uintptr_t)1023);
  plan(s, nullptr, true);
  if (s->ws_bytes > bytes) {
    delete s;
    return BB_ERR_NOMEM;
  }
  plan(s, base, false);
  s->ws = (char*)workspace;
  for (int i = 0; i < BB_VIEW_COUNT; ++i)
    if (s->layout[i][1]) s->layout[i][0] += (long long)(base - (char*)workspace);
  if (getenv("BB_KLOG") != nullptr && atoi(getenv("BB_KLOG")) != 0) {
    const int cap = 1 << 20;
    if (cudaMalloc(&s->klog, (1 + 2 * (size_t)cap) * 8) == cudaSuccess) {
      cudaMemset(s->klog, 0, 8);
      s->D.klog = s->klog;
      s->D.klog_cap = cap;
    }
  }
  rc = setup_gemms(s);
  if (rc != BB_OK) {
    delete s;
    return rc;
  }
  // static slot defaults (padding rows never change)
  std::vector<int> neg(std::max(s->blk.rows_alloc, s->full.rows_alloc), -1);
  std::vector<int> zero(neg.size(), 0);
  cudaMemcpy(s->blk.slot_pos, neg.data(), s->blk.rows_alloc * 4, cudaMemcpyHostToDevice);
  const int full_buf_rows = std::max(s->full.rows_alloc, s->fullr.rows_alloc);
  if ((int)neg.size() < full_buf_rows) neg.resize(full_buf_rows, -1);
  cudaMemcpy(s->full.slot_pos, neg.data(), (size_t)full_buf_rows * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(s->H.masked, zero.data(), s->blk.rows_alloc * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(s->full_rows, &s->S.NF, sizeof(int), cudaMemcpyHostToDevice);
  {
    const int nr = s->S.NF * s->S.B;
    cudaMemcpy(s->fullr_rows, &nr, sizeof(int), cudaMemcpyHostToDevice);
  }
  cudaMemset(s->st.init_gen, 0xFF, (size_t)s->S.R * s->S.G * 4);  // no presets: every position masked
  {
    std::vector<int> base(s->S.R);
    for (int r = 0; r < s->S.R; ++r) base[r] = r * s->S.NRq;
    cudaMemcpy(s->blk.req_base, base.data(), base.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(s->blk.rows_live, &s->S.NR, sizeof(int), cudaMemcpyHostToDevice);
  }
  {
    std::vector<unsigned long long> ts(17 * 8, 0ull);
    for (int k = 0; k < 16; ++k) ts[k * 8] = ~0ull;
    cudaMemcpy(s->tstat, ts.data(), ts.size() * 8, cudaMemcpyHostToDevice);
    std::vector<unsigned long long> site((size_t)3 * 10 * s->D.layers, 0ull);
    for (size_t i = 0; i < site.size(); i += 3) site[i] = site[i + 1] = ~0ull;
    cudaMemcpy(s->tsite, site.data(), site.size() * 8, cudaMemcpyHostToDevice);
  }
  if (cudaMallocHost(&s->host_ctrl, 4 * (size_t)s->S.R * C_WORDS * 4) != cudaSuccess) {
    delete s;
    return BB_ERR_CUDA;
  }
  for (int i = 0; i < 4; ++i) cudaEventCreateWithFlags(&s->ev[i], cudaEventDisableTiming);
  *out = s;
  return BB_OK;
}

BB_API int bb_session_destroy(void* sess) {
  Session* s = (Session*)sess;
  if (!s) return BB_OK;
  if (s->g_iter) cudaGraphExecDestroy(s->g_iter);
  if (s->g_iter_ref) cudaGraphExecDestroy(s->g_iter_ref);
  if (s->g_prefill) cudaGraphExecDestroy(s->g_prefill);
  if (s->g_vanilla) cudaGraphExecDestroy(s->g_vanilla);
  if (s->klog) cudaFree(s->klog);
  if (s->host_ctrl) cudaFreeHost(s->host_ctrl);
  for (int i = 0; i < 4; ++i)
    if (s->ev[i]) cudaEventDestroy(s->ev[i]);
  delete s;
  return BB_OK;
}

BB_API int bb_session_view(const void* sess, int which, long long* offset, long long* bytes) {
  const Session* s = (const Session*)sess;
  if (!s || which < 0 || which >= BB_VIEW_COUNT) return BB_ERR_CONTRACT;
  *offset = s->layout[which][0];
  *bytes = s->layout[which][1];
  return BB_OK;
}

BB_API int bb_session_info(const void* sess, int* out, int n) {
  const Session* s = (const Session*)sess;
  if (!s || !out) return BB_ERR_CONTRACT;
  int v[16] = {s->S.R, s->S.B, s->S.L, s->S.ev_cap, EVW, C_WORDS, B_WORDS, s->S.n_lp, s->S.pool,
               s->blk.rows_alloc, s->full.rows_alloc, s->gb.BN, s->gf.BN, s->S.max_items, s->S.NRq, s->S.ps};
  for (int i = 0; i < n && i < 16; ++i) out[i] = v[i];
  return BB_OK;
}

BB_API int bb_prefill(void* sess, void* stream) {
  Session* s = (Session*)sess;
  if (!s) return BB_ERR_CONTRACT;
  return enqueue_prefill(s, (cudaStream_t)stream);
}

BB_API int bb_block_step(void* sess, void* stream) {
  Session* s = (Session*)sess;
  if (!s) return BB_ERR_CONTRACT;
  return enqueue_block_step(s, (cudaStream_t)stream);
}

BB_API int bb_refresh(void* sess, void* stream) {
  Session* s = (Session*)sess;
  if (!s) return BB_ERR_CONTRACT;
  return enqueue_refresh(s, (cudaStream_t)stream);
}

BB_API int bb_iteration(void* sess, int with_refresh, int use_graph, void* stream) {
  Session* s = (Session*)sess;
  if (!s) return BB_ERR_CONTRACT;
  cudaStream_t st = (cudaStream_t)stream;
  if (!use_graph) {
    int rc = enqueue_block_step(s, st);
    if (rc == BB_OK && with_refresh) rc = enqueue_refresh(s, st);
    return rc;
  }
  cudaGraphExec_t* g = with_refresh ? &s->g_iter_ref : &s->g_iter;
  long long* nn = with_refresh ? &s->nodes_iter_ref : &s->nodes_iter;
  if (!*g) {
    int rc = capture(s, with_refresh ? 1 : 0, st, g, nn);
    if (rc != BB_OK) return rc;
  }
  CK(cudaGraphLaunch(*g, st));
  s->kernel_launches += *nn;
  s->graph_launches += 1;
  return BB_OK;
}

// Full run_blockbatch loop (scheduler.py:225-394) for every request of the
// session: prefill, then iterations until all requests finished (status 1) or
// failed (< 0).  Refresh is enqueued after every refresh_interval-th iteration
// (the device asserts that it matches its own counter).  Status words are
// polled asynchronously one iteration behind, so the host never stalls the
// GPU; the (at most one) extra iteration is a device-side no-op.
namespace {
struct NvtxRange {  // host-side range (enqueue + polling) of a bb_run phase
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

BB_API int bb_run(void* sess, int max_iterations, int use_graph, void* stream, int* iterations_out) {
  Session* s = (Session*)sess;
  if (!s) return BB_ERR_CONTRACT;
  NvtxRange run_range("bb_run");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = BB_OK;
  {
  NvtxRange prefill_range("bb_run:prefill");
  if (use_graph) {
    if (!s->g_prefill) {
      rc = capture(s, 2, st, &s->g_prefill, &s->nodes_prefill);
      if (rc != BB_OK) return rc;
    }
    CK(cudaGraphLaunch(s->g_prefill, st));
    s->kernel_launches += s->nodes_prefill;
    s->graph_launches += 1;
  } else {
    rc = enqueue_prefill(s, st);
    if (rc != BB_OK) return rc;
  }
  }
  const int R = s->S.R;
  const size_t cb = (size_t)R * C_WORDS * 4;
  CK(cudaMemcpyAsync(s->host_ctrl, s->st.ctrl, cb, cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(s->ev[0], st));
  int it = 0;
  bool finished = false;
  // status polled one iteration behind: while the host waits for iteration
  // it - 1, iteration it is already queued, so the GPU never idles and at most
  // one extra (no-op) iteration runs after the last request finished
  const int lag = 1;
  int checked = -1;
  while (!finished && it < max_iterations) {
    // check the status copied `lag` iterations ago
    const int chk = it - lag;
    if (chk >= 0 && chk > checked) {
      CK(cudaEventSynchronize(s->ev[chk & 3]));
      checked = chk;
      const int32_t* c = s->host_ctrl + (size_t)(chk & 3) * R * C_WORDS;
      finished = true;
      for (int r = 0; r < R; ++r) finished &= c[r * C_WORDS + C_STATUS] != 0;
      if (finished) break;
    }
    ++it;
    const bool with_refresh = it % s->S.refresh_interval == 0;
    NvtxRange it_range(with_refresh ? "bb_run:iteration+refresh" : "bb_run:iteration");
    rc = bb_iteration(s, with_refresh, use_graph, st);
    if (rc != BB_OK) return rc;
    CK(cudaMemcpyAsync(s->host_ctrl + (size_t)(it & 3) * R * C_WORDS, s->st.ctrl, cb, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(s->ev[it & 3], st));
  }
  CK(cudaStreamSynchronize(st));
  if (iterations_out) *iterations_out = it;
  return BB_OK;
}

BB_API int bb_prefill_part(void* sess, int part, void* stream) {
  Session* s = (Session*)sess;
  if (!s || part < 0 || part > 1) return BB_ERR_CONTRACT;
  return enqueue_prefill_part(s, part, (cudaStream_t)stream);
}

BB_API int bb_block_step_part(void* sess, int part, void* stream) {
  Session* s = (Session*)sess;
  if (!s || part < 0 || part > 2) return BB_ERR_CONTRACT;
  return enqueue_block_step_part(s, part, (cudaStream_t)stream);
}

BB_API int bb_kv_gather(void* sess, int r, int k, float* dst, void* stream) {
  Session* s = (Session*)sess;
  if (!s || !dst || r < 0 || r >= s->S.R || k < 0 || k >= s->S.B) return BB_ERR_CONTRACT;
  CK(launch_kv_gather(s->D, s->S, s->st, r, k, dst, (cudaStream_t)stream));
  return BB_OK;
}

// full_forward (model.py:322-328) of branch k's current row into the scratch
// pages, vectorized into dst; the branch's page table is restored afterwards
BB_API int bb_fresh_kv(void* sess, int r, int k, float* dst, void* stream) {
  Session* s = (Session*)sess;
  if (!s || !dst || r < 0 || r >= s->S.R || k < 0 || k >= s->S.B) return BB_ERR_CONTRACT;
  if (!s->S.diag) return fail(BB_ERR_CONFIG, "bb_fresh_kv needs a diagnostics session");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemsetAsync(s->full.skip, 1, sizeof(int), st));
  CK(launch_fresh_pack(s->D, s->S, s->st, s->full, r, k, s->fresh_save, st));
  CK(launch_attn_keys(s->D, s->S, s->full, s->st, st));
  CK(forward(s, s->full, s->gf, st));
  CK(launch_kv_gather(s->D, s->S, s->st, r, k, dst, st));
  CK(launch_fresh_restore(s->S, s->st, r, k, s->fresh_save, st));
  return BB_OK;
}

BB_API int bb_seam_init(void* sess, void* stream) {
  Session* s = (Session*)sess;
  if (!s || !s->desc.seam) return BB_ERR_CONTRACT;
  CK(launch_seam_init(s->D, s->S, s->st, (cudaStream_t)stream));
  return BB_OK;
}

BB_API int bb_seam_forward(void* sess, int full, int branch_mask, int use_target, void* stream) {
  Session* s = (Session*)sess;
  if (!s || !s->desc.seam || branch_mask <= 0 || branch_mask >= (1 << s->S.B)) return BB_ERR_CONTRACT;
  const Dims& D = s->D;
  const Sess& S = s->S;
  cudaStream_t st = (cudaStream_t)stream;
  if (!full) {
    CK(launch_seam_block_pack(D, S, s->st, s->blk, s->H, branch_mask, use_target, st));
    CK(launch_attn_keys(D, S, s->blk, s->st, st));
    CK(forward(s, s->blk, s->gb, st));
  } else {
    CK(cudaMemsetAsync(s->H.masked, 0, (size_t)s->blk.rows_alloc * 4, st));
    for (int k = 0; k < S.B; ++k) {
      if (!((branch_mask >> k) & 1)) continue;
      CK(launch_seam_full_pack(D, S, s->st, s->full, s->blk, s->H, k, use_target, st));
      CK(launch_attn_keys(D, S, s->full, s->st, st));
      CK(forward(s, s->full, s->gf, st));
      CK(launch_gather_head(D, S, s->full, s->blk, s->H, k, st));
    }
  }
  CK(head(s, st));
  return BB_OK;
}

BB_API int bb_kv_scatter(void* sess, int r, int k, const float* src, void* stream) {
  Session* s = (Session*)sess;
  if (!s || !src || r < 0 || r >= s->S.R || k < 0 || k >= s->S.B) return BB_ERR_CONTRACT;
  CK(launch_kv_scatter(s->D, s->S, s->st, r, k, src, (cudaStream_t)stream));
  return BB_OK;
}

BB_API int bb_head_logits(void* sess, float* logits, float* probs, void* stream) {
  Session* s = (Session*)sess;
  if (!s || !logits || !probs) return BB_ERR_CONTRACT;
  if (s->D.dtype == BB_DTYPE_BF16 && s->H.raw == nullptr) return fail(BB_ERR_CONFIG, "bb_head_logits needs desc.logits");
  CK(launch_head_logits(s->D, s->blk, s->H, logits, probs, (cudaStream_t)stream));
  return BB_OK;
}

BB_API int bb_sqdiff_norm(void* sess, const float* a, const float* b, long long n, double* out, void* stream) {
  Session* s = (Session*)sess;
  if (!s || !a || !out || n < 0) return BB_ERR_CONTRACT;
  CK(launch_sqdiff_norm(a, b, n, s->sq_part, s->n_sms, out, (cudaStream_t)stream));
  return BB_OK;
}

// vanilla_decode (decoding.py:279-321) for every request of a session with
// one branch of block size gen_len: initial rows, then rounds (one full
// forward each, captured once into a graph) until every request finished;
// status polled one round behind like bb_run.
BB_API int bb_run_vanilla(void* sess, int max_iterations, int use_graph, void* stream, int* iterations_out) {
  Session* s = (Session*)sess;
  if (!s) return BB_ERR_CONTRACT;
  if (s->S.B != 1 || s->S.bs[0] != s->S.G) return fail(BB_ERR_CONFIG, "vanilla: one branch of block size gen_len");
  cudaStream_t st = (cudaStream_t)stream;
  CK(launch_prefill_init(s->D, s->S, s->st, s->full, s->blk, s->H, st));
  const int R = s->S.R;
  const size_t cb = (size_t)R * C_WORDS * 4;
  // slot 0 = the initial state (the polling below reads slot (it - lag) & 3)
  CK(cudaMemcpyAsync(s->host_ctrl, s->st.ctrl, cb, cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(s->ev[0], st));
  int it = 0, checked = -1;
  bool finished = false;
  const int lag = 1;
  while (!finished && it < max_iterations) {
    const int chk = it - lag;
    if (chk >= 0 && chk > checked) {
      CK(cudaEventSynchronize(s->ev[chk & 3]));
      checked = chk;
      const int32_t* c = s->host_ctrl + (size_t)(chk & 3) * R * C_WORDS;
      finished = true;
      for (int r = 0; r < R; ++r) finished &= c[r * C_WORDS + C_STATUS] != 0;
      if (finished) break;
    }
    ++it;
    if (use_graph) {
      if (!s->g_vanilla) {
        const int rc = capture(s, 3, st, &s->g_vanilla, &s->nodes_vanilla);
        if (rc != BB_OK) return rc;
      }
      CK(cudaGraphLaunch(s->g_vanilla, st));
      s->kernel_launches += s->nodes_vanilla;
      s->graph_launches += 1;
    } else {
      const int rc = enqueue_vanilla(s, st);
      if (rc != BB_OK) return rc;
    }
    CK(cudaMemcpyAsync(s->host_ctrl + (size_t)(it & 3) * R * C_WORDS, s->st.ctrl, cb, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(s->ev[it & 3], st));
  }
  CK(cudaStreamSynchronize(st));
  if (iterations_out) *iterations_out = it;
  return BB_OK;
}

// live kernel timing: out[16][5] = (unused min, unused max, GEMM sum ns from the dependency-wait
// return, sum ns (GEMMs: from kernel entry), launches)
// kinds 0-3: block-pass QKV, O, gate/up, down; 4: LM head; 8-11: full-pass QKV..down;
// 5/13: block/full-pass tensor-core attention duration after its PDL wait,
// 6/14: spread of that attention's CTA start times (cluster placement)
BB_API int bb_session_gemm_stats(void* sess, unsigned long long* host_out, int reset, void* stream) {
  Session* s = (Session*)sess;
  if (!s || !host_out) return BB_ERR_CONTRACT;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<unsigned long long> ts(16 * 8);
  CK(cudaMemcpyAsync(ts.data(), s->tstat, ts.size() * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int k = 0; k < 16; ++k)
    for (int j = 0; j < 5; ++j) host_out[k * 5 + j] = ts[k * 8 + j];
  if (reset) {
    for (int k = 0; k < 16; ++k) {
      ts[k * 8 + 0] = ~0ull;
      for (int j = 1; j < 8; ++j) ts[k * 8 + j] = 0;
    }
    CK(cudaMemcpyAsync(s->tstat, ts.data(), ts.size() * 8, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  return BB_OK;
}

// timeline sessions (BB_KLOG=1): fused-QKV block attention phase offsets,
// out[8] = (CTAs, sum ns to: rows/keys loaded, phase-A loads issued, splice
// stored, cluster barrier, q gathered + chunk 0 landed, chunk loop done, end)
// out[8..15]: the BB_GPH_KIND GEMM's phase sums (GemmTcParams::ph)
BB_API int bb_session_phase_stats(void* sess, unsigned long long* out, int reset, void* stream) {
  Session* s = (Session*)sess;
  if (!s || !out) return BB_ERR_CONTRACT;
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(out, s->tstat + 7 * 8, 8 * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(out + 8, s->tstat + 16 * 8, 8 * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (reset) {
    CK(cudaMemsetAsync(s->tstat + 7 * 8, 0, 8 * 8, st));
    CK(cudaMemsetAsync(s->tstat + 16 * 8, 0, 8 * 8, st));
    CK(cudaStreamSynchronize(st));
  }
  return BB_OK;
}

// out[0] = kernel launches enqueued through graphs, [1] graph launches,
// [2] kernels per block-step graph, [3] per step+refresh graph, [4] per prefill graph
BB_API int bb_session_counters(void* sess, long long* out) {
  Session* s = (Session*)sess;
  if (!s || !out) return BB_ERR_CONTRACT;
  out[0] = s->kernel_launches;
  out[1] = s->graph_launches;
  out[2] = s->nodes_iter;
  out[3] = s->nodes_iter_ref;
  out[4] = s->nodes_prefill;
  return BB_OK;
}

// kernel timeline (BB_KLOG=1 sessions): copies up to `cap` (id, t_ns) pairs,
// returns the number recorded in *n (and resets the log if reset != 0)
BB_API int bb_session_klog(void* sess, unsigned long long* host_out, int cap, int reset, long long* n, void* stream) {
  Session* s = (Session*)sess;
  if (!s || !n) return BB_ERR_CONTRACT;
  cudaStream_t st = (cudaStream_t)stream;
  *n = 0;
  if (!s->klog) return BB_OK;
  unsigned long long cnt = 0;
  CK(cudaMemcpyAsync(&cnt, s->klog, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const long long m = (long long)(cnt < (unsigned long long)cap ? cnt : (unsigned long long)cap);
  if (host_out && m > 0) {
    CK(cudaMemcpyAsync(host_out, s->klog + 1, (size_t)m * 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  *n = m;
  if (reset) {
    CK(cudaMemsetAsync(s->klog, 0, 8, st));
    CK(cudaStreamSynchronize(st));
  }
  return BB_OK;
}

// host snapshot of the per-request control words (synchronous)
BB_API int bb_session_ctrl(void* sess, int* host_out, void* stream) {
  Session* s = (Session*)sess;
  if (!s || !host_out) return BB_ERR_CONTRACT;
  CK(cudaMemcpyAsync(host_out, s->st.ctrl, (size_t)s->S.R * C_WORDS * 4, cudaMemcpyDeviceToHost,
                     (cudaStream_t)stream));
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return BB_OK;
}

}  // extern "C"
