// STDiT3 step runtime behind the C ABI: model registration, request (shard geometry,
// workspace carve-up, text / cross-attention K/V cache, pre-built GEMM plans) and the
// denoise step as a fixed kernel sequence on one stream (capturable in a CUDA graph).
//
// Step (rank r of a DoP-P group):
//   begin : t / fps embedding -> t_block -> modulation table of all 2*depth blocks (+ final);
//           patch-embed + pos-embed of the local frames into x_sp [B][Tl][S][C] (fp32)
//   phase : for each block k: LN+mod -> QKV GEMM (+bias, q/k RMSNorm, RoPE) -> self-attn ->
//           proj GEMM (+gate, residual, bf16 copy) -> cross-q GEMM -> cross-attn -> out GEMM
//           (+residual) -> LN+mod -> fc1 GEMM (+GELU) -> fc2 GEMM (+gate, residual);
//           then (P > 1) push x to the other layout on every rank (sp->tp after spatial
//           blocks, tp->sp after temporal blocks) and barrier
//   end   : final LN+mod + Linear + unpatchify + CFG + Euler on the local frames of z
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <atomic>
#include <new>
#include <vector>

#include "capi_internal.h"
#include "common.cuh"
#include "elementwise.cuh"
#include "exchange.cuh"
#include "gemm_sm100.cuh"

#include "fmha_plan.cuh"
#include "temporal_plan.cuh"

using namespace ddit;
typedef __nv_bfloat16 bf16;

struct ddit_model {
  ddit_config cfg;
  ddit_weights w;
  std::vector<ddit_block_weights> blocks;
  const float** sst_dev = nullptr;  // device array of 2*depth scale_shift_table pointers
  // every block's cross-attention K/V projection stacked into one [2*depth*2C, C] matrix (+ bias)
  // so a request's whole K/V cache is ONE GEMM (M = B*300, N = 2*depth*2C = 129024 at XL/2)
  bf16* ckv_all = nullptr;
  float* ckv_b_all = nullptr;
  // every block's QKV weight with each head's 72 rows padded to an 80-row slot (8 zero rows) and
  // the bias likewise: the QKV GEMM then runs 256 x 240 tiles (3 whole heads, the per-head
  // RMSNorm / RoPE epilogue intact) instead of 256 x 144 -- shared-memory traffic per FLOP 178 ->
  // 131 B/clk; the padded columns are zeros and never stored
  bf16* qkv_pad = nullptr;
  float* qkv_bpad = nullptr;
};

namespace {
enum { G_QKV = 0, G_PROJ, G_CQ, G_CPROJ, G_FC1, G_FC2, G_N };

constexpr int kQkvSlot = 80;  // padded head slot of the QKV GEMM (rows of qkv_pad per head)

// dst row r of a [3 heads x 80] padded matrix <- src row (r / 80) * 72 + r % 80, zero if r % 80 >= 72
__global__ void qkv_pad_kernel(const bf16* __restrict__ w, const float* __restrict__ b,
                               bf16* __restrict__ wp, float* __restrict__ bp, int rows_pad, int C) {
  const int r = blockIdx.x;
  const int slot = r / kQkvSlot, j = r % kQkvSlot;
  const bool real = j < 72;
  const uint4* src = reinterpret_cast<const uint4*>(w + (size_t)(slot * 72 + (real ? j : 0)) * C);
  uint4* dst = reinterpret_cast<uint4*>(wp + (size_t)r * C);
  for (int i = threadIdx.x; i < C / 8; i += blockDim.x) dst[i] = real ? src[i] : make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) bp[r] = real ? b[slot * 72 + j] : 0.f;
}

int g_qkv_pad = -1;  // DDIT_QKV_PAD=0: the unpadded 144-column tiles
bool qkv_pad_enabled() {
  if (g_qkv_pad < 0) {
    const char* e = getenv("DDIT_QKV_PAD");
    g_qkv_pad = (e && e[0] == '0') ? 0 : 1;
  }
  return g_qkv_pad != 0;
}

struct Geometry {
  int B = 2;
  int T, Hl, Wl, h, w, S;
  int P, rank;
  int t_lo, t_hi, s_lo, s_hi, Tl, Sl;
  int M_sp, M_tp, Mmax;
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Carve {
  size_t off = 0;
  size_t take(size_t bytes) {
    size_t o = off;
    off = align256(off + bytes);
    return o;
  }
};

struct Layout {
  size_t x_sp, x_tp, xb, xm, big, ao, mods, fin, temb, tmlp, hbuf, freq, tv, pos, rope, yemb, kv,
      flags, counter, total;
};

int geometry(const ddit_config& c, const ddit_req_desc& d, Geometry* g) {
  if (d.dop < 1 || d.dop > kMaxDop || (d.dop & (d.dop - 1)) || d.rank < 0 || d.rank >= d.dop) {
    set_error("dop %d / rank %d invalid (dop must be a power of two <= %d)", d.dop, d.rank,
              kMaxDop);
    return DDIT_E_LOOKUP;
  }
  if (d.latent_t <= 0 || d.latent_h <= 0 || d.latent_w <= 0 || d.num_steps <= 0) {
    set_error("bad request shape");
    return DDIT_E_INVALID;
  }
  g->T = d.latent_t;
  g->Hl = d.latent_h;
  g->Wl = d.latent_w;
  g->h = (d.latent_h + 1) / 2;
  g->w = (d.latent_w + 1) / 2;
  g->S = g->h * g->w;
  g->P = d.dop;
  g->rank = d.rank;
  const int tc = (g->T + g->P - 1) / g->P, sc = (g->S + g->P - 1) / g->P;
  g->t_lo = std::min(d.rank * tc, g->T);
  g->t_hi = std::min((d.rank + 1) * tc, g->T);
  g->s_lo = std::min(d.rank * sc, g->S);
  g->s_hi = std::min((d.rank + 1) * sc, g->S);
  g->Tl = g->t_hi - g->t_lo;
  g->Sl = g->s_hi - g->s_lo;
  g->M_sp = g->B * g->Tl * g->S;
  g->M_tp = g->B * g->T * g->Sl;
  g->Mmax = std::max(g->M_sp, g->M_tp);
  (void)c;
  return DDIT_OK;
}

Layout layout(const ddit_config& c, const Geometry& g) {
  Layout L;
  Carve cv;
  const size_t C = c.hidden;
  const size_t Ly = (size_t)g.B * c.text_tokens;
  const size_t nblk = 2 * (size_t)c.depth;
  L.x_sp = cv.take((size_t)std::max(g.M_sp, 1) * C * 4);
  L.x_tp = g.P > 1 ? cv.take((size_t)std::max(g.M_tp, 1) * C * 4) : L.x_sp;
  L.xb = cv.take((size_t)g.Mmax * C * 2);
  L.xm = cv.take((size_t)g.Mmax * C * 2);
  size_t big = std::max((size_t)g.Mmax * std::max((size_t)c.mlp_hidden, 3 * C),
                        Ly * (size_t)c.caption_channels + Ly * C);
  L.big = cv.take(big * 2);
  L.ao = cv.take((size_t)g.Mmax * C * 2);
  L.mods = cv.take(nblk * g.B * 6 * C * 4);
  L.fin = cv.take((size_t)g.B * 2 * C * 4);
  L.temb = cv.take((size_t)g.B * C * 4);
  L.tmlp = cv.take((size_t)g.B * 6 * C * 4);
  L.hbuf = cv.take((size_t)g.B * C * 4);
  L.freq = cv.take((size_t)2 * g.B * c.freq_dim * 4);
  L.tv = cv.take(4096 * 4);
  L.pos = cv.take((size_t)g.S * C * 4);
  L.rope = cv.take((size_t)g.T * c.head_dim * 4);
  L.yemb = cv.take(Ly * C * 2);
  L.kv = cv.take(nblk * Ly * 2 * C * 2);
  L.flags = cv.take(kMaxDop * 4);
  L.counter = cv.take(16);
  L.total = cv.off;
  return L;
}

}  // namespace

struct ddit_req {
  ddit_model* m;
  ddit_req_desc d;
  Geometry g;
  Layout L;
  uint8_t* ws;
  float *x_sp, *x_tp, *mods, *fin, *temb, *tmlp, *hbuf, *freq, *tv, *pos, *rope;
  bf16 *xb, *xm, *big, *ao, *yemb, *kv;
  uint32_t* flags;
  unsigned int* counter;
  std::vector<float> ts;  // transformed timesteps
  std::vector<GemmPlan> plans;  // [2*depth][G_N]
  std::vector<GemmPlan> text_plans;  // y_embedder fc1, fc2, then the 2*depth cross K/V GEMMs
  std::vector<FmhaPlan> fm_self;   // [2*depth] tcgen05 self-attention plans (spatial blocks)
  std::vector<FmhaPlan> fm_cross;  // [2*depth] tcgen05 cross-attention plans
  std::vector<uint8_t> fm_self_ok, fm_cross_ok;
  std::vector<TemporalPlan> tm_self;  // [2*depth] tcgen05 temporal-attention plans (T <= 32)
  std::vector<uint8_t> tm_self_ok;
  PeerPtrs peer_sp{}, peer_tp{};
  PeerFlags peer_flags{};
  bool peers_set = false;
  bool flags_set = false;
  bool fused_xch = false;        // the fc2 GEMM of every block performs the DSP exchange
  bool external_xch = false;     // the caller moves the rows (staged pack -> ncclAllToAll -> unpack)
  // profiling: event pairs around every launch, tagged by kernel class
  bool prof_on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<int> ev_cls;
  size_t ev_n = 0;
  int device = 0;                           // the GPU this rank state lives on
  cudaEvent_t rs0 = nullptr, rs1 = nullptr;  // timing of the last re-shard into this rank
  ~ddit_req() {
    for (auto e : ev) cudaEventDestroy(e);
    if (rs0) cudaEventDestroy(rs0);
    if (rs1) cudaEventDestroy(rs1);
  }
};

static std::atomic<unsigned long long> g_launches{0};

// GEMM -> exchange fusion for DoP > 1 (env DDIT_FUSED_XCH=0 / ddit_set_fused_exchange(0): the
// separate exchange kernel), read when a request's peers are registered
static int g_fused_xch = -1;
static bool fused_exchange_enabled() {
  if (g_fused_xch < 0) {
    const char* e = getenv("DDIT_FUSED_XCH");
    g_fused_xch = (e && e[0] == '0') ? 0 : 1;
  }
  return g_fused_xch != 0;
}

namespace {
enum { K_GEMM = 0, K_ATTN = 1, K_EW = 2, K_EXCH = 3, K_NCLASS = 4 };

// Run `f` (which launches kernels on s and returns 0 / a DDIT_E code) counting `n` launches
// and, when profiling, bracketing it with a pair of events of class `cls`.
template <class F>
int timed(ddit_req* r, int cls, cudaStream_t s, int n, F&& f) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (r->prof_on) {
    while (r->ev.size() < 2 * (r->ev_n + 1)) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) break;
      r->ev.push_back(e);
    }
    if (r->ev.size() >= 2 * (r->ev_n + 1)) {
      e0 = r->ev[2 * r->ev_n];
      e1 = r->ev[2 * r->ev_n + 1];
      if (r->ev_cls.size() <= r->ev_n) r->ev_cls.resize(r->ev_n + 1);
      r->ev_cls[r->ev_n] = cls;
      r->ev_n++;
      cudaEventRecord(e0, s);
    }
  }
  int rc = f();
  if (e1) cudaEventRecord(e1, s);
  g_launches += (unsigned long long)n;
  return rc;
}
}  // namespace

namespace {

// RFLOW timesteps with the OpenSora-1.2 resolution/length transform (oracle/stdit3.py).
std::vector<float> rflow_timesteps(const ddit_req_desc& d) {
  std::vector<float> out(d.num_steps);
  const double ratio = std::sqrt((double)d.height * d.width / (512.0 * 512.0)) *
                       std::sqrt((double)d.latent_t);
  for (int i = 0; i < d.num_steps; ++i) {
    const double u = 1.0 - (double)i / d.num_steps;
    out[i] = (float)(ratio * u / (1.0 + (ratio - 1.0) * u) * 1000.0);
  }
  return out;
}

float step_dt(const ddit_req* r, int step) {
  const auto& ts = r->ts;
  const double dt = step < (int)ts.size() - 1 ? (double)ts[step] - ts[step + 1] : ts[step];
  return (float)(dt / 1000.0);
}

int pick_bn(int n) {
  for (int bn : {192, 256, 128, 96})
    if (n % bn == 0) return bn;
  return 0;
}

// block GEMM plan with the tile chosen for this rank's M (gemm_pick_tile)
int plan_auto(GemmPlan* p, const void* A, int lda, const void* B, int ldb, int M, int N, int K,
              int epi, const EpiParams& e) {
  int bn = 0, two = 0;
  gemm_pick_tile(M, N, epi, &bn, &two);
  return gemm_plan_init_cta(p, A, lda, B, ldb, M, N, K, epi, e, bn, two);
}

int build_plans(ddit_req* r) {
  const ddit_config& c = r->m->cfg;
  const Geometry& g = r->g;
  const int C = c.hidden;
  const int nblk = 2 * c.depth;
  r->plans.assign((size_t)nblk * G_N, GemmPlan{});
  for (int k = 0; k < nblk; ++k) {
    const bool temporal = k & 1;
    const int M = temporal ? g.M_tp : g.M_sp;
    if (M == 0) continue;
    float* x = temporal ? r->x_tp : r->x_sp;
    const int rpb = M / g.B;
    const ddit_block_weights& bw = r->m->blocks[k];
    const float* mod = r->mods + (size_t)k * g.B * 6 * C;
    GemmPlan* P = &r->plans[(size_t)k * G_N];
    EpiParams e;
    int rc;
    // QKV: bias + q/k RMSNorm (+ RoPE over frames for temporal blocks)
    memset(&e, 0, sizeof e);
    e.bias = bw.qkv_b;
    e.out = r->big;
    e.ldo = 3 * C;
    e.qnorm_w = bw.q_norm;
    e.knorm_w = bw.k_norm;
    e.hidden = C;
    e.rope = temporal ? 1 : 0;
    e.rope_T = g.T;
    e.rope_S = temporal ? g.Sl : g.S;
    e.rope_tab = reinterpret_cast<const float2*>(r->rope);
    e.eps = c.eps;
    e.rows_per_b = rpb;
    if (r->m->qkv_pad && qkv_pad_enabled()) {
      const int rows_pad = 3 * c.heads * kQkvSlot;
      e.bias = r->m->qkv_bpad + (size_t)k * rows_pad;
      if ((rc = gemm_plan_init_cta(&P[G_QKV], r->xm, C, r->m->qkv_pad + (size_t)k * rows_pad * C, C, M,
                                   rows_pad, C, EPI_QKV, e, 240, two_cta_enabled() ? 1 : 0)))
        return rc;
    } else if ((rc = plan_auto(&P[G_QKV], r->xm, C, bw.qkv_w, C, M, 3 * C, C, EPI_QKV, e))) {
      return rc;
    }
    // attention out-projection: x += gate_msa * (.) ; bf16 copy of x for cross-attn queries
    memset(&e, 0, sizeof e);
    e.bias = bw.proj_b;
    e.resid = x;
    e.ldr = C;
    e.gate = mod + 2 * C;
    e.gate_stride = 6 * C;
    e.rows_per_b = rpb;
    e.out2 = r->xb;
    e.ldo2 = C;
    if ((rc = plan_auto(&P[G_PROJ], r->ao, C, bw.proj_w, C, M, C, C, EPI_RESID, e)))
      return rc;
    // cross-attn queries
    memset(&e, 0, sizeof e);
    e.bias = bw.cq_b;
    e.out = r->xm;
    e.ldo = C;
    e.rows_per_b = rpb;
    if ((rc = plan_auto(&P[G_CQ], r->xb, C, bw.cq_w, C, M, C, C, EPI_BF16, e))) return rc;
    // cross-attn out projection: x += (.)
    memset(&e, 0, sizeof e);
    e.bias = bw.cproj_b;
    e.resid = x;
    e.ldr = C;
    e.rows_per_b = rpb;
    if ((rc = plan_auto(&P[G_CPROJ], r->ao, C, bw.cproj_w, C, M, C, C, EPI_RESID, e)))
      return rc;
    // MLP
    memset(&e, 0, sizeof e);
    e.bias = bw.fc1_b;
    e.out = r->big;
    e.ldo = c.mlp_hidden;
    e.rows_per_b = rpb;
    if ((rc = plan_auto(&P[G_FC1], r->xm, C, bw.fc1_w, C, M, c.mlp_hidden, C, EPI_GELU_BF16, e)))
      return rc;
    memset(&e, 0, sizeof e);
    e.bias = bw.fc2_b;
    e.resid = x;
    e.ldr = C;
    e.gate = mod + 5 * C;
    e.gate_stride = 6 * C;
    e.rows_per_b = rpb;
    if ((rc = plan_auto(&P[G_FC2], r->big, c.mlp_hidden, bw.fc2_w, c.mlp_hidden, M, C,
                        c.mlp_hidden, EPI_RESID, e)))
      return rc;
  }
  return DDIT_OK;
}

int launch(const GemmPlan& p, cudaStream_t s) {
  int rc = gemm_plan_launch(&p, s);
  if (rc) {
    set_error("gemm: %s", gemm_last_error());
    return DDIT_E_CUDA;
  }
  return DDIT_OK;
}

int launch_g(ddit_req* r, const GemmPlan& p, cudaStream_t s) {
  return timed(r, K_GEMM, s, 1, [&] { return launch(p, s); });
}
int ln_mod(ddit_req* r, float* x, int M, const float* shift, const float* scale, int rpb,
           cudaStream_t s) {
  const ddit_config& c = r->m->cfg;
  return timed(r, K_EW, s, 1, [&] {
    if (ln_modulate(x, r->xm, M, c.hidden, shift, scale, 6 * c.hidden, rpb, c.eps, s)) {
      set_error("ln_modulate: bad shape");
      return (int)DDIT_E_INVALID;
    }
    return (int)DDIT_OK;
  });
}
// Temporal self-attention runs the tcgen05 plan built at request open (T <= 64 latent frames,
// i.e. every OpenSora clip length); there is no other kernel for it on the step path.
int attn_temporal(ddit_req* r, int k, const ddit_attn* a, cudaStream_t s) {
  (void)a;
  if (!r->tm_self_ok[k]) {
    set_error("block %d: temporal attention plan missing (T <= 64 latent frames supported)", k);
    return DDIT_E_CONFIG;
  }
  const TemporalPlan& tp = r->tm_self[k];
  return timed(r, K_ATTN, s, 1, [&] { return temporal_plan_launch(&tp, s); });
}

// Self-attention index map of block k (spatial: frames are sequences; temporal: positions).
ddit_attn self_attn_args(const ddit_req* r, int k) {
  const ddit_config& c = r->m->cfg;
  const Geometry& g = r->g;
  const int C = c.hidden;
  ddit_attn a;
  memset(&a, 0, sizeof a);
  a.q = r->big;
  a.k = r->big + C;
  a.v = r->big + 2 * C;
  a.ldq = a.ldk = a.ldv = 3 * C;
  a.o = r->ao;
  a.ldo = C;
  a.heads = c.heads;
  a.head_dim = c.head_dim;
  a.scale = 1.0f / std::sqrt((float)c.head_dim);
  if (!(k & 1)) {
    a.num_seqs = g.B * g.Tl;
    a.Lq = a.Lk = g.S;
    a.q_inner = a.kv_inner = 1;
    a.q_outer = a.kv_outer = g.S;
    a.q_tok = a.kv_tok = 1;
  } else {
    a.num_seqs = g.B * g.Sl;
    a.Lq = a.Lk = g.T;
    a.q_inner = a.kv_inner = g.Sl;
    a.q_outer = a.kv_outer = g.T * g.Sl;
    a.q_inner_stride = a.kv_inner_stride = 1;
    a.q_tok = a.kv_tok = g.Sl;
  }
  return a;
}

// Cross attention of block k: each batch's rows attend to its own 300 text tokens.
ddit_attn cross_attn_args(const ddit_req* r, int k) {
  const ddit_config& c = r->m->cfg;
  const Geometry& g = r->g;
  const int C = c.hidden;
  const int M = (k & 1) ? g.M_tp : g.M_sp;
  const int rpb = M / g.B;
  // kv [B*300][2*depth][2C]: block k's K at column 2Ck, its V at 2Ck + C
  const bf16* kv = r->kv + (size_t)k * 2 * C;
  ddit_attn a;
  memset(&a, 0, sizeof a);
  a.q = r->xm;
  a.ldq = C;
  a.k = kv;
  a.v = kv + C;
  a.ldk = a.ldv = 2 * c.depth * 2 * C;
  a.o = r->ao;
  a.ldo = C;
  a.heads = c.heads;
  a.head_dim = c.head_dim;
  a.num_seqs = g.B;
  a.Lq = rpb;
  a.Lk = c.text_tokens;
  a.q_inner = a.kv_inner = 1;
  a.q_outer = rpb;
  a.kv_outer = c.text_tokens;
  a.q_tok = a.kv_tok = 1;
  a.scale = 1.0f / std::sqrt((float)c.head_dim);
  return a;
}

int build_attn_plans(ddit_req* r) {
  const int nblk = 2 * r->m->cfg.depth;
  r->fm_self.assign(nblk, FmhaPlan{});
  r->fm_cross.assign(nblk, FmhaPlan{});
  r->fm_self_ok.assign(nblk, 0);
  r->fm_cross_ok.assign(nblk, 0);
  r->tm_self.assign(nblk, TemporalPlan{});
  r->tm_self_ok.assign(nblk, 0);
  for (int k = 0; k < nblk; ++k) {
    const int M = (k & 1) ? r->g.M_tp : r->g.M_sp;
    if (M == 0) continue;
    ddit_attn a = self_attn_args(r, k);
    if (!(k & 1) && fmha_supported(&a)) {
      int rc = fmha_plan_init(&r->fm_self[k], &a);
      if (rc) return rc;
      r->fm_self_ok[k] = 1;
    }
    if (k & 1) {  // T > 64 latent frames: the request cannot open (no other temporal kernel)
      int rc = temporal_plan_init(&r->tm_self[k], &a);
      if (rc) return rc;
      r->tm_self_ok[k] = 1;
    }
    a = cross_attn_args(r, k);
    if (fmha_supported(&a)) {
      int rc = fmha_plan_init(&r->fm_cross[k], &a);
      if (rc) return rc;
      r->fm_cross_ok[k] = 1;
    }
  }
  return DDIT_OK;
}

// Spatial and cross attention run the tcgen05 FMHA plan built at request open; there is no
// other kernel for them on the step path (a layout the plan cannot take fails the step).
// Temporal self-attention (T <= 32 keys per sequence) has its own kernel.
int run_attn(ddit_req* r, int k, bool cross, cudaStream_t s) {
  if (!cross && (k & 1)) {
    ddit_attn a = self_attn_args(r, k);
    return attn_temporal(r, k, &a, s);
  }
  const std::vector<uint8_t>& ok = cross ? r->fm_cross_ok : r->fm_self_ok;
  if (!ok[k]) {
    set_error("block %d: %s attention layout not supported by the tcgen05 FMHA", k,
              cross ? "cross" : "spatial");
    return DDIT_E_CONFIG;
  }
  const FmhaPlan& fp = cross ? r->fm_cross[k] : r->fm_self[k];
  return timed(r, K_ATTN, s, 1, [&] { return fmha_plan_launch(&fp, s); });
}

int run_block(ddit_req* r, int k, cudaStream_t s) {
  const ddit_config& c = r->m->cfg;
  const Geometry& g = r->g;
  const int C = c.hidden;
  const bool temporal = k & 1;
  const int M = temporal ? g.M_tp : g.M_sp;
  if (M == 0) return DDIT_OK;
  const int rpb = M / g.B;
  float* x = temporal ? r->x_tp : r->x_sp;
  const float* mod = r->mods + (size_t)k * g.B * 6 * C;
  const GemmPlan* P = &r->plans[(size_t)k * G_N];
  int rc;
  if ((rc = ln_mod(r, x, M, mod + 0 * C, mod + 1 * C, rpb, s))) return rc;
  if ((rc = launch_g(r, P[G_QKV], s))) return rc;
  if ((rc = run_attn(r, k, false, s))) return rc;
  if ((rc = launch_g(r, P[G_PROJ], s))) return rc;
  if ((rc = launch_g(r, P[G_CQ], s))) return rc;
  if ((rc = run_attn(r, k, true, s))) return rc;
  if ((rc = launch_g(r, P[G_CPROJ], s))) return rc;
  if ((rc = ln_mod(r, x, M, mod + 3 * C, mod + 4 * C, rpb, s))) return rc;
  if ((rc = launch_g(r, P[G_FC1], s))) return rc;
  if ((rc = launch_g(r, P[G_FC2], s))) return rc;
  return DDIT_OK;
}

int push_exchange(ddit_req* r, int k, cudaStream_t s) {
  const Geometry& g = r->g;
  if (g.P == 1 || r->external_xch) return DDIT_OK;
  // fused: the block's fc2 GEMM already stored its rows at their owners and signalled (a rank
  // without rows in this layout runs no GEMM, so it still signals through the exchange kernel)
  if (r->fused_xch && ((k & 1) ? g.M_tp : g.M_sp) > 0) return DDIT_OK;
  if (!r->peers_set) {
    set_error("DoP %d request has no peers registered", g.P);
    return DDIT_E_CONFIG;
  }
  const int C = r->m->cfg.hidden;
  ExchangeSync sync;
  memset(&sync, 0, sizeof sync);
  if (r->flags_set) {
    sync.flags = r->peer_flags;
    sync.counter = r->counter;
    sync.epoch = r->counter + 1;
    sync.rank = g.rank;
    sync.P = g.P;
  }
  int n = 0;
  timed(r, K_EXCH, s, 0, [&] {
    if ((k & 1) == 0)
      n = exchange_sp_to_tp(r->x_sp, r->peer_tp, g.B, g.T, g.S, C, g.P, g.t_lo, g.Tl, sync, s);
    else
      n = exchange_tp_to_sp(r->x_tp, r->peer_sp, g.B, g.T, g.S, C, g.P, g.s_lo, g.Sl, sync, s);
    return 0;
  });
  g_launches += (unsigned long long)n;
  return check_cuda("exchange");
}

}  // namespace

extern "C" {

DDIT_API int ddit_model_create(const ddit_config* cfg, const ddit_weights* w, ddit_model** out) {
  if (!cfg || !w || !out || !w->blocks) {
    set_error("ddit_model_create: null argument");
    return DDIT_E_INVALID;
  }
  if (cfg->head_dim != 72 || cfg->heads * cfg->head_dim != cfg->hidden ||
      cfg->hidden % 144 != 0 || cfg->in_channels * 4 > 16) {
    set_error("ddit_model_create: unsupported config (head_dim 72, C %% 144 == 0 required)");
    return DDIT_E_CONFIG;
  }
  ddit_model* m = new (std::nothrow) ddit_model();
  if (!m) return DDIT_E_ALLOC;
  m->cfg = *cfg;
  m->w = *w;
  m->blocks.assign(w->blocks, w->blocks + 2 * cfg->depth);
  m->w.blocks = nullptr;
  std::vector<const float*> sst(2 * cfg->depth);
  for (int k = 0; k < 2 * cfg->depth; ++k) sst[k] = m->blocks[k].scale_shift_table;
  if (cudaMalloc(&m->sst_dev, sst.size() * sizeof(float*)) != cudaSuccess ||
      cudaMemcpy(m->sst_dev, sst.data(), sst.size() * sizeof(float*), cudaMemcpyHostToDevice) !=
          cudaSuccess) {
    set_error("ddit_model_create: cudaMalloc failed");
    ddit_model_destroy(m);
    return DDIT_E_ALLOC;
  }
  // stacked cross-attention K/V weights (a device-side copy; the caller's tensors stay theirs)
  const size_t kvw = (size_t)2 * cfg->hidden * cfg->hidden, kvb = (size_t)2 * cfg->hidden;
  bool ok = cudaMalloc(&m->ckv_all, 2 * cfg->depth * kvw * sizeof(bf16)) == cudaSuccess &&
            cudaMalloc(&m->ckv_b_all, 2 * cfg->depth * kvb * sizeof(float)) == cudaSuccess;
  for (int k = 0; ok && k < 2 * cfg->depth; ++k)
    ok = cudaMemcpy(m->ckv_all + k * kvw, m->blocks[k].ckv_w, kvw * sizeof(bf16),
                    cudaMemcpyDeviceToDevice) == cudaSuccess &&
         cudaMemcpy(m->ckv_b_all + k * kvb, m->blocks[k].ckv_b, kvb * sizeof(float),
                    cudaMemcpyDeviceToDevice) == cudaSuccess;
  if (!ok) {
    set_error("ddit_model_create: stacked K/V weights: %s", cudaGetErrorString(cudaGetLastError()));
    ddit_model_destroy(m);
    return DDIT_E_ALLOC;
  }
  const int rows_pad = 3 * cfg->heads * kQkvSlot;
  ok = cudaMalloc(&m->qkv_pad, (size_t)2 * cfg->depth * rows_pad * cfg->hidden * sizeof(bf16)) == cudaSuccess &&
       cudaMalloc(&m->qkv_bpad, (size_t)2 * cfg->depth * rows_pad * sizeof(float)) == cudaSuccess;
  for (int k = 0; ok && k < 2 * cfg->depth; ++k) {
    qkv_pad_kernel<<<rows_pad, 128>>>(static_cast<const bf16*>(m->blocks[k].qkv_w), m->blocks[k].qkv_b,
                                      m->qkv_pad + (size_t)k * rows_pad * cfg->hidden,
                                      m->qkv_bpad + (size_t)k * rows_pad, rows_pad, cfg->hidden);
    ok = cudaGetLastError() == cudaSuccess;
  }
  if (!ok || cudaDeviceSynchronize() != cudaSuccess) {
    set_error("ddit_model_create: padded QKV weights: %s", cudaGetErrorString(cudaGetLastError()));
    ddit_model_destroy(m);
    return DDIT_E_ALLOC;
  }
  *out = m;
  return DDIT_OK;
}

DDIT_API int ddit_set_qkv_pad(int on) {
  g_qkv_pad = on ? 1 : 0;
  return DDIT_OK;
}

DDIT_API void ddit_model_destroy(ddit_model* m) {
  if (!m) return;
  cudaFree(m->sst_dev);
  cudaFree(m->ckv_all);
  cudaFree(m->ckv_b_all);
  cudaFree(m->qkv_pad);
  cudaFree(m->qkv_bpad);
  delete m;
}

DDIT_API int ddit_request_workspace_bytes(const ddit_model* m, const ddit_req_desc* d,
                                          uint64_t* bytes) {
  Geometry g;
  int rc = geometry(m->cfg, *d, &g);
  if (rc) return rc;
  *bytes = layout(m->cfg, g).total;
  return DDIT_OK;
}

DDIT_API int ddit_request_shard(const ddit_model* m, const ddit_req_desc* d, int* t_lo, int* t_hi,
                                int* s_lo, int* s_hi) {
  Geometry g;
  ddit_config none;
  memset(&none, 0, sizeof none);
  int rc = geometry(m ? m->cfg : none, *d, &g);  // pure host math: model may be NULL
  if (rc) return rc;
  *t_lo = g.t_lo;
  *t_hi = g.t_hi;
  *s_lo = g.s_lo;
  *s_hi = g.s_hi;
  return DDIT_OK;
}

// Caption -> per-request text state: [y_cond; y_null] -> bf16 -> y_embedder MLP -> yemb
// [B*300, C], then the per-block cross-attention K/V cache kv[k] = yemb . Wkv^T + b.
// The 2 + 2*depth GEMM plans (fixed buffers of the request) are built once per request, so
// re-binding a pooled request or rebuilding the K/V cache after a promotion costs only launches.
static int text_plans(ddit_req* r) {
  if (!r->text_plans.empty()) return DDIT_OK;
  const ddit_model* m = r->m;
  const ddit_config& c = m->cfg;
  const int Ly = r->g.B * c.text_tokens;
  bf16* ycat = r->big;
  bf16* yhid = r->big + (size_t)Ly * c.caption_channels;
  std::vector<GemmPlan> tp(3);
  EpiParams e;
  memset(&e, 0, sizeof e);
  e.bias = m->w.y1_b;
  e.out = yhid;
  e.ldo = c.hidden;
  if (gemm_plan_init(&tp[0], ycat, c.caption_channels, m->w.y1_w, c.caption_channels, Ly, c.hidden,
                     c.caption_channels, EPI_GELU_BF16, e, pick_bn(c.hidden))) {
    set_error("y_embedder fc1 plan: %s", gemm_last_error());
    return DDIT_E_INVALID;
  }
  e.bias = m->w.y2_b;
  e.out = r->yemb;
  if (gemm_plan_init(&tp[1], yhid, c.hidden, m->w.y2_w, c.hidden, Ly, c.hidden, c.hidden, EPI_BF16,
                     e, pick_bn(c.hidden))) {
    set_error("y_embedder fc2 plan: %s", gemm_last_error());
    return DDIT_E_INVALID;
  }
  // all blocks' K/V in one GEMM: kv [Ly][2*depth*2C] = yemb . ckv_all^T + ckv_b_all
  const int nkv = 2 * c.depth * 2 * c.hidden;
  memset(&e, 0, sizeof e);
  e.bias = m->ckv_b_all;
  e.out = r->kv;
  e.ldo = nkv;
  int bn = 0, two = 0;
  gemm_pick_tile(Ly, nkv, EPI_BF16, &bn, &two);
  if (gemm_plan_init_cta(&tp[2], r->yemb, c.hidden, m->ckv_all, c.hidden, Ly, nkv, c.hidden,
                         EPI_BF16, e, bn, two)) {
    set_error("cross kv plan: %s", gemm_last_error());
    return DDIT_E_INVALID;
  }
  r->text_plans.swap(tp);
  return DDIT_OK;
}

// per-block cross-attention K/V cache from the request's yemb
static int cross_kv(ddit_req* r, cudaStream_t s) {
  int rc = text_plans(r);
  if (rc) return rc;
  if ((rc = launch(r->text_plans[2], s))) return rc;
  g_launches += 1;
  return DDIT_OK;
}

static int embed_text(ddit_req* r, const float* y_cond, cudaStream_t s) {
  const ddit_model* m = r->m;
  const ddit_config& c = m->cfg;
  int rc = text_plans(r);
  if (rc) return rc;
  const size_t ycount = (size_t)c.text_tokens * c.caption_channels;
  bf16* ycat = r->big;
  cast_bf16(y_cond, ycat, ycount, s);
  cast_bf16(m->w.y_null, ycat + ycount, ycount, s);
  if ((rc = launch(r->text_plans[0], s)) || (rc = launch(r->text_plans[1], s))) return rc;
  g_launches += 4;
  if ((rc = cross_kv(r, s))) return rc;
  return check_cuda("embed_text");
}

DDIT_API int ddit_request_open(ddit_model* m, const ddit_req_desc* d, void* workspace,
                               uint64_t bytes, const float* y_cond, void* stream, ddit_req** out) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ddit_req* r = new (std::nothrow) ddit_req();
  if (!r) return DDIT_E_ALLOC;
  r->m = m;
  r->d = *d;
  cudaGetDevice(&r->device);
  int rc = geometry(m->cfg, *d, &r->g);
  if (rc) {
    delete r;
    return rc;
  }
  r->L = layout(m->cfg, r->g);
  if (bytes < r->L.total || (reinterpret_cast<uintptr_t>(workspace) & 255)) {
    set_error("workspace too small or misaligned (%llu < %llu)", (unsigned long long)bytes,
              (unsigned long long)r->L.total);
    delete r;
    return DDIT_E_ALLOC;
  }
  const ddit_config& c = m->cfg;
  const Geometry& g = r->g;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  r->ws = ws;
  r->x_sp = reinterpret_cast<float*>(ws + r->L.x_sp);
  r->x_tp = reinterpret_cast<float*>(ws + r->L.x_tp);
  r->xb = reinterpret_cast<bf16*>(ws + r->L.xb);
  r->xm = reinterpret_cast<bf16*>(ws + r->L.xm);
  r->big = reinterpret_cast<bf16*>(ws + r->L.big);
  r->ao = reinterpret_cast<bf16*>(ws + r->L.ao);
  r->mods = reinterpret_cast<float*>(ws + r->L.mods);
  r->fin = reinterpret_cast<float*>(ws + r->L.fin);
  r->temb = reinterpret_cast<float*>(ws + r->L.temb);
  r->tmlp = reinterpret_cast<float*>(ws + r->L.tmlp);
  r->hbuf = reinterpret_cast<float*>(ws + r->L.hbuf);
  r->freq = reinterpret_cast<float*>(ws + r->L.freq);
  r->tv = reinterpret_cast<float*>(ws + r->L.tv);
  r->pos = reinterpret_cast<float*>(ws + r->L.pos);
  r->rope = reinterpret_cast<float*>(ws + r->L.rope);
  r->yemb = reinterpret_cast<bf16*>(ws + r->L.yemb);
  r->kv = reinterpret_cast<bf16*>(ws + r->L.kv);
  r->flags = reinterpret_cast<uint32_t*>(ws + r->L.flags);
  r->counter = reinterpret_cast<unsigned int*>(ws + r->L.counter);
  r->ts = rflow_timesteps(*d);
  if (d->num_steps > 1000) {
    set_error("num_steps too large");
    delete r;
    return DDIT_E_INVALID;
  }
  // timestep table tv[step][4] = {t, t, fps, fps}
  std::vector<float> tv((size_t)d->num_steps * 4);
  for (int i = 0; i < d->num_steps; ++i) {
    tv[4 * i + 0] = tv[4 * i + 1] = r->ts[i];
    tv[4 * i + 2] = tv[4 * i + 3] = d->fps;
  }
  cudaMemcpyAsync(r->tv, tv.data(), tv.size() * 4, cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(r->flags, 0, kMaxDop * 4, s);
  cudaMemsetAsync(r->counter, 0, 16, s);
  // tables
  const int base_size = (int)std::lround(std::sqrt((double)g.S));
  const float scale = (float)(std::sqrt((double)d->height * d->width) / c.input_sq_size);
  build_tables(r->pos, g.h, g.w, c.hidden, scale, (float)base_size, r->rope, g.T, c.head_dim, s);
  if ((rc = embed_text(r, y_cond, s))) {
    delete r;
    return rc;
  }
  if ((rc = build_plans(r))) {
    set_error("plan: %s", gemm_last_error());
    delete r;
    return rc == -3 ? DDIT_E_TMA : DDIT_E_INVALID;
  }
  if ((rc = build_attn_plans(r))) {
    delete r;
    return rc;
  }
  if ((rc = check_cuda("ddit_request_open"))) {
    delete r;
    return rc;
  }
  *out = r;
  return DDIT_OK;
}

DDIT_API void ddit_request_close(ddit_req* r) { delete r; }

// On failure the request stays open and owned by the caller (its text state is undefined until
// a later set_text / copy_text succeeds); it is never freed here.
DDIT_API int ddit_request_set_text(ddit_req* r, const float* y_cond, void* stream) {
  if (!r || !y_cond) {
    set_error("ddit_request_set_text: null argument");
    return DDIT_E_INVALID;
  }
  return embed_text(r, y_cond, static_cast<cudaStream_t>(stream));
}

DDIT_API int ddit_request_copy_text(ddit_req* dst, const ddit_req* src, void* stream) {
  const ddit_config& c = dst->m->cfg;
  if (src->m->cfg.hidden != c.hidden || src->m->cfg.depth != c.depth ||
      src->m->cfg.text_tokens != c.text_tokens || src->g.B != dst->g.B) {
    set_error("copy_text: requests of different models");
    return DDIT_E_CONFIG;
  }
  const size_t Ly = (size_t)dst->g.B * c.text_tokens;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // plain UVA copies: peer-to-peer over NVLink when src lives on another (peer-enabled) device
  cudaMemcpyAsync(dst->yemb, src->yemb, Ly * c.hidden * 2, cudaMemcpyDefault, s);
  cudaMemcpyAsync(dst->kv, src->kv, (size_t)2 * c.depth * Ly * 2 * c.hidden * 2, cudaMemcpyDefault, s);
  return check_cuda("ddit_request_copy_text");
}

// Promotion-time text state for a new rank: only the y-embedding (B*300 x C bf16, 1.4 MB at XL/2)
// crosses from src (a peer copy when src is on another device); the 2*depth cross-attention K/V
// projections are recomputed on dst's own GPU (bit-identical: same kernels, same inputs), so a
// 1 -> 8 promotion does not push 8 x 155 MB of K/V cache out of one GPU.
DDIT_API int ddit_request_share_text(ddit_req* dst, const ddit_req* src, void* stream) {
  if (!dst || !src) {
    set_error("ddit_request_share_text: null argument");
    return DDIT_E_INVALID;
  }
  const ddit_config& c = dst->m->cfg;
  if (src->m->cfg.hidden != c.hidden || src->m->cfg.depth != c.depth ||
      src->m->cfg.text_tokens != c.text_tokens || src->g.B != dst->g.B) {
    set_error("share_text: requests of different models");
    return DDIT_E_CONFIG;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t Ly = (size_t)dst->g.B * c.text_tokens;
  if (dst->yemb != src->yemb &&
      cudaMemcpyAsync(dst->yemb, src->yemb, Ly * c.hidden * 2, cudaMemcpyDefault, s) != cudaSuccess)
    return check_cuda("share_text copy");
  int rc = cross_kv(dst, s);
  if (rc) return rc;
  return check_cuda("ddit_request_share_text");
}

// Promotion P -> P' in one call (SURVEY.md §8(b) `ddit_reshard`; reference engine.py:281-290
// charges OverheadModel's 1 ms broadcast + 1 ms scale-up): for every rank i of the new group, on
// its own device and stream, gather its new T-shard of z from the old group's shards (peer
// loads) and take the text state from text_src (ddit_request_share_text). Host cost is one call
// for the whole group; each new rank records start / end events (ddit_request_reshard_ms).
DDIT_API int ddit_reshard(ddit_req* const* new_ranks, float* const* new_z, int q,
                          const float* const* old_z, const int* old_t_lo, const int* old_t_hi,
                          int p, const ddit_req* text_src, void* const* streams) {
  if (!new_ranks || !new_z || !old_z || !old_t_lo || !old_t_hi || !text_src || q < 1 ||
      q > kMaxDop || p < 1 || p > kMaxDop) {
    set_error("ddit_reshard: bad arguments");
    return DDIT_E_INVALID;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  int rc = DDIT_OK;
  for (int i = 0; i < q && rc == DDIT_OK; ++i) {
    ddit_req* r = new_ranks[i];
    cudaStream_t s = streams ? static_cast<cudaStream_t>(streams[i]) : nullptr;
    cudaSetDevice(r->device);
    if (!r->rs0 && (cudaEventCreate(&r->rs0) != cudaSuccess || cudaEventCreate(&r->rs1) != cudaSuccess)) {
      rc = check_cuda("reshard events");
      break;
    }
    cudaEventRecord(r->rs0, s);
    const ddit_config& c = r->m->cfg;
    rc = ddit_latent_gather(new_z[i], r->g.t_lo, r->g.t_hi, old_z, old_t_lo, old_t_hi, p,
                            c.in_channels, r->g.Hl * r->g.Wl, s);
    if (rc == DDIT_OK && r != text_src) rc = ddit_request_share_text(r, text_src, s);
    cudaEventRecord(r->rs1, s);
    g_launches += 1;
  }
  cudaSetDevice(prev);
  return rc;
}

DDIT_API int ddit_request_reshard_ms(ddit_req* r, float* ms) {
  if (!r || !ms || !r->rs0) {
    set_error("ddit_request_reshard_ms: no re-shard recorded");
    return DDIT_E_INVALID;
  }
  if (cudaEventSynchronize(r->rs1) != cudaSuccess ||
      cudaEventElapsedTime(ms, r->rs0, r->rs1) != cudaSuccess)
    return check_cuda("ddit_request_reshard_ms");
  return DDIT_OK;
}

DDIT_API int ddit_request_exchange_buffers(ddit_req* r, void** x_sp, void** x_tp, void** flags) {
  *x_sp = r->x_sp;
  *x_tp = r->x_tp;
  *flags = r->flags;
  return DDIT_OK;
}

DDIT_API int ddit_request_set_peers(ddit_req* r, void* const* x_sp, void* const* x_tp,
                                    void* const* flags) {
  for (int q = 0; q < r->g.P; ++q) {
    r->peer_sp.p[q] = static_cast<float*>(x_sp[q]);
    r->peer_tp.p[q] = static_cast<float*>(x_tp[q]);
    r->peer_flags.p[q] = flags ? static_cast<uint32_t*>(flags[q]) : nullptr;
  }
  r->peers_set = true;
  r->flags_set = flags != nullptr;
  // GEMM -> exchange fusion: every block's fc2 plan stores its rows at their owner rank
  const Geometry& g = r->g;
  r->fused_xch = g.P > 1 && fused_exchange_enabled();
  for (int k = 0; k < 2 * r->m->cfg.depth && !r->plans.empty(); ++k) {
    GemmPlan& fc2 = r->plans[(size_t)k * G_N + G_FC2];
    EpiParams& e = fc2.ep;
    e.xch = 0;
    if (!r->fused_xch) {
      gemm_plan_refresh(&fc2);
      continue;
    }
    const bool temporal = k & 1;
    e.xch = temporal ? 2 : 1;
    for (int q = 0; q < kMaxDop; ++q) {
      e.xdst[q] = q < g.P ? (temporal ? r->peer_sp.p[q] : r->peer_tp.p[q]) : nullptr;
      e.xflags[q] = q < g.P && r->flags_set ? r->peer_flags.p[q] : nullptr;
    }
    e.xB = g.B;
    e.xT = g.T;
    e.xS = g.S;
    e.xP = g.P;
    e.xlo = temporal ? g.s_lo : g.t_lo;
    e.xlen = temporal ? g.Sl : g.Tl;
    e.xchunk = temporal ? (g.T + g.P - 1) / g.P : (g.S + g.P - 1) / g.P;
    e.xcounter = r->counter;
    e.xepoch = r->counter + 1;
    e.xrank = g.rank;
    gemm_plan_refresh(&fc2);  // the exchange epilogue has no wide tile
  }
  return DDIT_OK;
}

DDIT_API int ddit_request_timestep(const ddit_req* r, int step, float* t, float* dt) {
  if (step < 0 || step >= r->d.num_steps) {
    set_error("step %d outside [0, %d)", step, r->d.num_steps);
    return DDIT_E_INVALID;
  }
  *t = r->ts[step];
  *dt = step_dt(r, step);
  return DDIT_OK;
}

DDIT_API int ddit_step_begin(ddit_req* r, const float* z_local, int step, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (step < 0 || step >= r->d.num_steps) {
    set_error("step %d outside [0, %d)", step, r->d.num_steps);
    return DDIT_E_INVALID;
  }
  const ddit_model* m = r->m;
  const ddit_config& c = m->cfg;
  const ddit_weights& w = m->w;
  const Geometry& g = r->g;
  const int C = c.hidden, B = g.B;
  // t / fps embedding -> t (temb) -> t_block (tmlp)
  return timed(r, K_EW, s, 8, [&] {
  timestep_freq(r->freq, r->tv + 4 * step, 2 * B, c.freq_dim, s);
  const float* ft = r->freq;
  const float* ff = r->freq + (size_t)B * c.freq_dim;
  gemv(static_cast<const bf16*>(w.t0_w), w.t0_b, ft, r->hbuf, B, C, c.freq_dim, 0, 1, 0, s);
  gemv(static_cast<const bf16*>(w.t2_w), w.t2_b, r->hbuf, r->temb, B, C, C, 0, 0, 0, s);
  gemv(static_cast<const bf16*>(w.f0_w), w.f0_b, ff, r->hbuf, B, C, c.freq_dim, 0, 1, 0, s);
  gemv(static_cast<const bf16*>(w.f2_w), w.f2_b, r->hbuf, r->temb, B, C, C, 0, 0, 1, s);
  gemv(static_cast<const bf16*>(w.tb_w), w.tb_b, r->temb, r->tmlp, B, 6 * C, C, 1, 0, 0, s);
  modulation(r->mods, m->sst_dev, r->tmlp, 2 * c.depth, B, C, r->fin, w.final_sst, r->temb, s);
  patch_embed(z_local, w.x_emb_w, w.x_emb_b, r->pos, r->x_sp, g.Tl, g.Hl, g.Wl, g.h, g.w, C,
              c.in_channels, B, s);
  return check_cuda("ddit_step_begin");
  });
}

DDIT_API int ddit_step_phase(ddit_req* r, int phase, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (phase < 0 || phase >= 2 * r->m->cfg.depth) {
    set_error("phase %d out of range", phase);
    return DDIT_E_INVALID;
  }
  int rc = run_block(r, phase, s);
  if (rc) return rc;
  if ((rc = check_cuda("block"))) return rc;
  return push_exchange(r, phase, s);
}

DDIT_API int ddit_step_barrier(ddit_req* r, void* stream) {
  if (r->g.P == 1) return DDIT_OK;
  if (!r->peers_set || !r->flags_set) {
    set_error("barrier: flags of the group not registered");
    return DDIT_E_CONFIG;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  timed(r, K_EXCH, s, 1, [&] {
    return flag_wait(r->flags, r->counter + 1, r->g.P, r->counter + 2, s);
  });
  return check_cuda("barrier");
}

DDIT_API int ddit_set_exchange_timeout_ms(int ms) {
  set_flag_timeout_ms(ms);
  return DDIT_OK;
}

DDIT_API int ddit_set_fused_exchange(int on) {
  g_fused_xch = on ? 1 : 0;
  return DDIT_OK;
}

DDIT_API int ddit_request_set_option(ddit_req* r, int option, int value) {
  switch (option) {
    case DDIT_OPT_TC_ATTENTION:  // retired: the step has one attention path (tcgen05 FMHA)
      if (value != 0) return DDIT_OK;
      set_error("DDIT_OPT_TC_ATTENTION=0 is no longer supported: the step always runs the tcgen05 FMHA");
      return DDIT_E_INVALID;
    case DDIT_OPT_EXTERNAL_XCH:
      r->external_xch = value != 0;
      return DDIT_OK;
  }
  set_error("unknown option %d", option);
  return DDIT_E_INVALID;
}

// ---- staged all-to-all for an external collective (the NCCL arm, DDIT_OPT_EXTERNAL_XCH)
static XchGeom xch_geom(const ddit_req* r) {
  const Geometry& g = r->g;
  XchGeom x;
  x.B = g.B;
  x.T = g.T;
  x.S = g.S;
  x.C = r->m->cfg.hidden;
  x.P = g.P;
  x.Tl = g.Tl;
  x.Sl = g.Sl;
  return x;
}

DDIT_API int ddit_request_xch_counts(ddit_req* r, int phase, int* send_rows, int* recv_rows) {
  if (!r || !send_rows || !recv_rows || phase < 0 || phase >= 2 * r->m->cfg.depth) {
    set_error("ddit_request_xch_counts: bad argument");
    return DDIT_E_INVALID;
  }
  xch_counts(xch_geom(r), phase & 1, send_rows, recv_rows);
  return DDIT_OK;
}

DDIT_API int ddit_request_xch_pack(ddit_req* r, int phase, void* send, void* stream) {
  if (!r || phase < 0 || phase >= 2 * r->m->cfg.depth) {
    set_error("ddit_request_xch_pack: bad argument");
    return DDIT_E_INVALID;
  }
  const XchGeom x = xch_geom(r);
  const int dir = phase & 1;
  int sr[kMaxDop], rr[kMaxDop], rows = 0;
  xch_counts(x, dir, sr, rr);
  for (int q = 0; q < x.P; ++q) rows += sr[q];
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int n = 0;
  timed(r, K_EXCH, s, 0, [&] {
    n = xch_pack(dir == 0 ? r->x_sp : r->x_tp, static_cast<float*>(send), x, dir, rows, s);
    return 0;
  });
  g_launches += (unsigned long long)n;
  return check_cuda("xch_pack");
}

DDIT_API int ddit_request_xch_unpack(ddit_req* r, int phase, const void* recv, void* stream) {
  if (!r || phase < 0 || phase >= 2 * r->m->cfg.depth) {
    set_error("ddit_request_xch_unpack: bad argument");
    return DDIT_E_INVALID;
  }
  const XchGeom x = xch_geom(r);
  const int dir = phase & 1;
  int sr[kMaxDop], rr[kMaxDop], rows = 0;
  xch_counts(x, dir, sr, rr);
  for (int q = 0; q < x.P; ++q) rows += rr[q];
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int n = 0;
  timed(r, K_EXCH, s, 0, [&] {
    n = xch_unpack(static_cast<const float*>(recv), dir == 0 ? r->x_tp : r->x_sp, x, dir, rows, s);
    return 0;
  });
  g_launches += (unsigned long long)n;
  return check_cuda("xch_unpack");
}

DDIT_API int ddit_request_profile(ddit_req* r, int enable) {
  r->prof_on = enable != 0;
  r->ev_n = 0;
  return DDIT_OK;
}

DDIT_API int ddit_request_profile_read(ddit_req* r, float* ms, int* count) {
  for (int c = 0; c < K_NCLASS; ++c) {
    ms[c] = 0.f;
    count[c] = 0;
  }
  if (r->ev_n == 0) return DDIT_OK;
  if (cudaEventSynchronize(r->ev[2 * r->ev_n - 1]) != cudaSuccess) return check_cuda("profile");
  for (size_t i = 0; i < r->ev_n; ++i) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r->ev[2 * i], r->ev[2 * i + 1]) != cudaSuccess)
      return check_cuda("profile elapsed");
    ms[r->ev_cls[i]] += t;
    count[r->ev_cls[i]] += 1;
  }
  r->ev_n = 0;
  return DDIT_OK;
}

// counter[0] = exchange CTA tickets, [1] = exchange epoch, [2] = barrier status (0 = ok,
// 1 + q = the wait on rank q's flag timed out: the group is broken)
DDIT_API int ddit_request_status(ddit_req* r, void* stream, uint32_t* status) {
  if (!r || !status) {
    set_error("ddit_request_status: null argument");
    return DDIT_E_INVALID;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t v = 0;
  if (cudaMemcpyAsync(&v, r->counter + 2, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return check_cuda("ddit_request_status");
  *status = v;
  if (v) {
    set_error("exchange barrier timed out waiting for rank %u of the group", v - 1);
    return DDIT_E_CONFIG;
  }
  return DDIT_OK;
}

DDIT_API unsigned long long ddit_launch_count(void) { return g_launches.load(); }

DDIT_API int ddit_step_end(ddit_req* r, float* z_local, int step, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const ddit_model* m = r->m;
  const ddit_config& c = m->cfg;
  const Geometry& g = r->g;
  return timed(r, K_EW, s, 1, [&] {
    if (final_layer(r->x_sp, r->fin, m->w.final_w, m->w.final_b, z_local, g.Tl, g.Hl, g.Wl, g.h,
                    g.w, c.hidden, c.in_channels, c.out_channels, r->d.guidance, step_dt(r, step),
                    c.eps, s)) {
      set_error("final layer: unsupported channel count");
      return (int)DDIT_E_CONFIG;
    }
    return check_cuda("ddit_step_end");
  });
}

DDIT_API int ddit_dit_step(ddit_req* r, float* z_local, int step, void* stream) {
  int rc = ddit_step_begin(r, z_local, step, stream);
  if (rc) return rc;
  for (int k = 0; k < 2 * r->m->cfg.depth; ++k) {
    if ((rc = ddit_step_phase(r, k, stream))) return rc;
    if ((rc = ddit_step_barrier(r, stream))) return rc;
  }
  return ddit_step_end(r, z_local, step, stream);
}

}  // extern "C"
