// Persistent warp-specialised tcgen05 GEMM for sm_100a with the STDiT epilogues fused.
//
//   warp 0      : TMA producer (one elected lane) -- A/B k-blocks into a STAGES-deep smem ring
//   warp 1      : MMA issuer   (one elected lane) -- tcgen05.mma 128xBNx16 into TMEM
//   warp 2      : TMEM allocator (512 columns: two accumulator buffers at columns 0 / 256)
//   warps 4..7  : epilogue -- tcgen05.ld (one accumulator row per thread) -> fused op ->
//                 swizzled smem staging -> TMA store (fp32 residual: TMA load, update, TMA store)
//
// The accumulator is double-buffered in TMEM so the epilogue of tile i overlaps the MMAs of
// tile i+1. The epilogue never issues per-row global stores: every output leaves through a
// TMA bulk tensor store from a 128 B-swizzled (bank-conflict-free) staging buffer, double
// buffered so the store of sub-tile s overlaps the math of sub-tile s+1.
// Shapes in the DDiT step: M = tokens (ragged; TMA zero-fills the
// M and K tails on load and clips on store), K in {288, 1152, 4096, 4608}, N % BN == 0.
#include "common.cuh"
#include "gemm_sm100.cuh"
#include "cta_pair.cuh"

#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>

namespace ddit {

static constexpr int BM = 128;
static constexpr int BK = 64;
static constexpr int kThreads = 256;
static constexpr int kTmemCols = 512;
static constexpr int kAccStride = 256;  // TMEM column offset of accumulator buffer 1

__host__ __device__ constexpr bool is_resid(int epi) {
  return epi == EPI_RESID || epi == EPI_RESID_COPY || epi == EPI_RESID_RED;
}

#ifndef DDIT_RSLOTS
#define DDIT_RSLOTS 2
#endif
#ifndef DDIT_RED_BUFS
#define DDIT_RED_BUFS 2
#endif
// DDIT_EPI_TRACE (experiment builds only): SM-clock timestamps of CTA 0's MMA issuer and first
// epilogue warp per tile / sub-tile, read back with ddit_debug_trace()
#ifdef DDIT_EPI_TRACE
__device__ unsigned long long g_epi_trace[1024];
#define EPI_TRACE(idx) \
  do {                 \
    if (blockIdx.x == 0) g_epi_trace[(idx) & 1023] = clock64(); \
  } while (0)
#else
#define EPI_TRACE(idx) \
  do {                 \
  } while (0)
#endif
template <int BN, int EPI>
struct EpiCfg {
  // staging bytes (two buffers) and sub-tile width (columns) per epilogue kind: bf16 outputs
  // use 64-column sub-tiles (128 B swizzle) when BN allows, else 32 (64 B swizzle)
  static constexpr bool BF = EPI == EPI_BF16 || EPI == EPI_GELU_BF16;
  // QKV: one head per sub-tile, in 72-column slots (BN 144) or 80-column padded slots (BN 240)
  static constexpr int SUB = EPI == EPI_QKV ? (BN == 240 ? 80 : 72) : BF ? (BN % 64 == 0 ? 64 : 32) : 32;
  static constexpr int BUF = EPI == EPI_QKV ? 128 * 144 : 128 * 128;  // main staging buffer
  // gated residual: each epilogue warp runs its own ring of RSLOTS fp32 32x32 sub-tiles (loads run
  // RSLOTS-2 sub-tiles ahead) + three bf16 copy buffers (SW64): WARP_BYTES per warp
  static constexpr bool RED = EPI == EPI_RESID_RED;
  static constexpr int RSLOTS = is_resid(EPI) ? (RED ? DDIT_RED_BUFS : DDIT_RSLOTS) : 0;
  // R >= 3: stores of sub-tile s-1 may still read while s runs (3 bf16 buffers, loads R-2 ahead);
  // R == 2: they must finish first (2 bf16 buffers, loads 1 ahead)
  static constexpr int RAHEAD = RSLOTS >= 3 ? RSLOTS - 2 : 1;
  static constexpr int NOB = RSLOTS >= 3 ? 3 : 2;
  // EPI_RESID_COPY: the bf16 copy of a PAIR of sub-tiles (32 rows x 64 cols, 128 B rows) leaves
  // in one TMA store -- 64 B-row boxes store at a fraction of the bandwidth
  static constexpr int OB = EPI == EPI_RESID_COPY ? 4096 : 2048;
  // EPI_RESID with BN % 64 == 0 never has a bf16 copy (the plan turns out2 into EPI_RESID_COPY),
  // so its copy buffers are not allocated: the smem goes back to the mainloop (fc2: 6 stages)
  static constexpr bool HAS_OB = EPI == EPI_RESID_COPY || (EPI == EPI_RESID && BN % 64 != 0);
  // EPI_RESID_RED: RSLOTS staging buffers per warp, each a 32 x 32 fp32 sub-tile on its way out
  // through a TMA reduce-add (no loads, no bf16 copy)
  static constexpr int WARP_BYTES = RSLOTS * 4096 + (HAS_OB ? NOB * OB : 0);
  // gated residual: the bias row and the B gate rows (all N columns) staged once per CTA, so the
  // per-sub-tile column vectors are shared-memory broadcasts instead of cold L2 reads (consecutive
  // tiles of a CTA have different column blocks)
  // QKV: bias. Plain epilogues keep __ldg: staging their bias cost 1.3 ms per 144p step (small-M
  // GEMMs have one or two tiles per CTA, so the per-CTA staging is not amortised)
  // sized to the XL/2 need (3 x 1152 or 3456 floats = 13.5 KB), so QKV keeps 7 mainloop stages
  static constexpr int COL_BYTES = is_resid(EPI) ? 13824 : EPI == EPI_QKV ? (BN == 240 ? 15360 : 13824) : 0;
  static constexpr int BYTES = is_resid(EPI) ? 4 * WARP_BYTES + COL_BYTES : 2 * BUF + COL_BYTES;
};
static constexpr int kRBars = 4 * 5;  // residual ring barriers (per warp) in the barrier block

template <int BN, int EPI>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_BYTES = 512;
  static constexpr int BUDGET = 232448 - 1024 - BAR_BYTES - EpiCfg<BN, EPI>::BYTES;
  static constexpr int STAGES_RAW = BUDGET / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + EpiCfg<BN, EPI>::BYTES + BAR_BYTES;
  static_assert(B_BYTES % 1024 == 0, "B tile must keep 1024 B swizzle-atom alignment");
  static_assert(BN % 16 == 0 && BN <= 256, "invalid UMMA N");
  static_assert(BN % EpiCfg<BN, EPI>::SUB == 0, "BN must be a multiple of the epilogue sub-tile");
  static_assert(STAGES >= (DDIT_RSLOTS > 2 ? 2 : 3), "pipeline too shallow");
};

DDIT_DEV void tmem_ld_32x32b_x8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
DDIT_DEV void tmem_ld_x32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

DDIT_DEV void tma_store_2d(const void* tmap, const void* smem_src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
               : "memory");
}
DDIT_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
DDIT_DEV void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
DDIT_DEV void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
DDIT_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
DDIT_DEV void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// 16-byte chunk j of row r in a 128 B-swizzled (Swizzle<3,4,3>) / 64 B-swizzled tile
DDIT_DEV uint32_t sw128(int r, int j) { return (uint32_t)(r * 128 + ((j ^ (r & 7)) << 4)); }
DDIT_DEV uint32_t sw64(int r, int j) { return (uint32_t)(r * 64 + ((j ^ ((r >> 1) & 3)) << 4)); }

DDIT_DEV void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
DDIT_DEV float4 ld_shared_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

DDIT_DEV float gelu_fast(float x) {
  // tanh-approximated GELU with the hardware tanh (MUFU.TANH); |err| << bf16 ulp
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return 0.5f * x * (1.0f + t);
}

struct EpiCtx {
  int m_tiles, n_tiles, num_tiles;
  int M, N;
};

// Stage bias[N] and gate[b][N] (b < ceil(M / rows_per_b)) into sCol (COL_BYTES) with the 128
// epilogue threads; returns sCol, or nullptr when they do not fit (the epilogue then reads them
// from global memory). Ends with the epilogue warps' named barrier.
template <int COL_BYTES>
DDIT_DEV const float* epi_stage_cols(const EpiParams& ep, float* sCol, int M, int N, int tid) {
  const int nb = ep.gate ? (M + ep.rows_per_b - 1) / ep.rows_per_b : 0;
  const bool fits = (size_t)(1 + nb) * N * 4 <= (size_t)COL_BYTES;
  if (fits) {  // all loads first (independent, one latency), then the shared stores
    constexpr int PER = COL_BYTES / 4 / 128;
    const int total = (1 + nb) * N;
    float v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int idx = tid + 128 * k;
      const int row = idx / N, col = idx - row * N;
      v[k] = idx >= total ? 0.f
             : row == 0   ? (ep.bias ? __ldg(ep.bias + col) : 0.f)
                          : __ldg(ep.gate + (size_t)(row - 1) * ep.gate_stride + col);
    }
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (tid + 128 * k < total) sCol[tid + 128 * k] = v[k];
  }
  epi_bar();
  return fits ? sCol : nullptr;
}

// The sequence of 128x32 residual sub-tiles this CTA's epilogue consumes: sub-tile j belongs to
// the CTA's (j / NS)-th tile (tile0 + i * tstride) at column block j % NS.
struct ResidStream {
  int tile0, tstride, num_tiles, n_tiles, mstep, moff;
  DDIT_DEV bool coord(int j, int ns, int& m0, int& c0) const {
    const int t = tile0 + (j / ns) * tstride;
    if (t >= num_tiles) return false;
    m0 = (t / n_tiles) * mstep + moff;
    c0 = (t % n_tiles) * (ns * 32) + (j % ns) * 32;
    return true;
  }
};

// Pull the i-th residual tile (this CTA's 128 rows x BN) of the stream into L2 ahead of its
// epilogue; tmP is a box-{BN, 128} map of the residual (no swizzle, L2 prefetch only).
template <int BN>
DDIT_DEV void resid_prefetch_l2(const ResidStream& rs, int i, const CUtensorMap* tmP) {
  int m0, c0;
  if (rs.coord(i * (BN / 32), BN / 32, m0, c0))
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(tmP)),
                 "r"(c0), "r"(m0)
                 : "memory");
}

// the same for a wide tile (2BN columns): both BN halves
template <int BN>
DDIT_DEV void resid_prefetch_l2_wide(const ResidStream& rs, int i, const CUtensorMap* tmP) {
  int m0, c0;
  if (rs.coord(i * (2 * BN / 32), 2 * BN / 32, m0, c0))
#pragma unroll
    for (int h = 0; h < 2; ++h)
      asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                       reinterpret_cast<uint64_t>(tmP)),
                   "r"(c0 + h * BN), "r"(m0)
                   : "memory");
}

// load residual sub-tile j of this warp's 32-row slab into ring slot j % R (wbase: the warp's
// ring, wbar: its R barriers)
template <int R>
DDIT_DEV void resid_issue(const ResidStream& rs, int ns, int j, int row_off, const CUtensorMap* tmR,
                          uint8_t* wbase, uint64_t* wbar) {
  int m0, c0;
  if (rs.coord(j, ns, m0, c0)) {
    const int slot = j % R;
    mbar_arrive_expect_tx(&wbar[slot], 4096);
    tma_load_2d(wbase + slot * 4096, tmR, &wbar[slot], c0, m0 + row_off);
  }
}

// ------------------------------------------------------------------ epilogue: bf16 / gelu / f32
template <int BN, int EPI>
DDIT_DEV void epi_plain_tile(const EpiParams& ep, const CUtensorMap* tmO, uint8_t* sE,
                             uint32_t taddr, int rit, int m0, int n0, bool elected, int& cnt,
                             uint32_t tempty_cl, int lane, const float* sCol) {
  constexpr int SUB = EpiCfg<BN, EPI>::SUB;
  constexpr int NS = BN / SUB;
#pragma unroll 1
  for (int sub = 0; sub < NS; ++sub) {
    uint8_t* sb = sE + (cnt & 1) * EpiCfg<BN, EPI>::BUF;
    const uint32_t sbase = smem_u32(sb);
    if (elected) bulk_wait_read<1>();
    epi_bar();
    uint32_t r[SUB];
    tmem_ld_x32(taddr + sub * SUB, r);
    if constexpr (SUB == 64) tmem_ld_x32(taddr + sub * SUB + 32, r + 32);
    tmem_ld_wait();
    if (sub == NS - 1) {  // accumulator fully read: hand TMEM back to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 31) mbar_arrive_cl_relaxed(tempty_cl);
    }
    const int col0 = n0 + sub * SUB;
    float v[SUB];
#pragma unroll
    for (int q = 0; q < SUB / 4; ++q) {
      float4 b = sCol     ? reinterpret_cast<const float4*>(sCol + col0)[q]
                 : ep.bias ? __ldg(reinterpret_cast<const float4*>(ep.bias + col0) + q)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      v[4 * q + 0] = __uint_as_float(r[4 * q + 0]) + b.x;
      v[4 * q + 1] = __uint_as_float(r[4 * q + 1]) + b.y;
      v[4 * q + 2] = __uint_as_float(r[4 * q + 2]) + b.z;
      v[4 * q + 3] = __uint_as_float(r[4 * q + 3]) + b.w;
    }
    if constexpr (EPI == EPI_GELU_BF16) {
#pragma unroll
      for (int e = 0; e < SUB; ++e) v[e] = gelu_fast(v[e]);
    }
    if constexpr (EPI == EPI_F32) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        st_shared_v4(sbase + sw128(rit, j), __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                     __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
    } else if constexpr (SUB == 32) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        st_shared_v4(sbase + sw64(rit, j), pack_bf16(v[8 * j], v[8 * j + 1]),
                     pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                     pack_bf16(v[8 * j + 6], v[8 * j + 7]));
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        st_shared_v4(sbase + sw128(rit, j), pack_bf16(v[8 * j], v[8 * j + 1]),
                     pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                     pack_bf16(v[8 * j + 6], v[8 * j + 7]));
    }
    fence_async_smem();
    epi_bar();
    if (elected) {
      tma_store_2d(tmO, sb, col0, m0);
      bulk_commit();
    }
    ++cnt;
  }
}

// ------------------------------------------------------------------ epilogue: gated residual
// Destination of row `row` (of this rank's layout) in its owner rank's other-layout buffer.
DDIT_DEV float* xch_row(const EpiParams& ep, int row, int C) {
  if (ep.xch == 1) {  // x_sp [B][Tl][S] -> x_tp of rank q [B][T][Sl_q]
    const int s = row % ep.xS, tl = (row / ep.xS) % ep.xlen, b = row / (ep.xS * ep.xlen);
    const int q = s / ep.xchunk, s_lo = q * ep.xchunk;
    const int Sl = min(s_lo + ep.xchunk, ep.xS) - s_lo;
    return ep.xdst[q] + (((size_t)b * ep.xT + ep.xlo + tl) * Sl + (s - s_lo)) * C;
  }
  // x_tp [B][T][Sl] -> x_sp of rank q [B][Tl_q][S]
  const int sl = row % ep.xlen, t = (row / ep.xlen) % ep.xT, b = row / (ep.xlen * ep.xT);
  const int q = t / ep.xchunk, t_lo = q * ep.xchunk;
  const int Tlq = min(t_lo + ep.xchunk, ep.xT) - t_lo;
  return ep.xdst[q] + (((size_t)b * Tlq + (t - t_lo)) * ep.xS + ep.xlo + sl) * C;
}

// End of a fused-exchange GEMM: after every CTA's stores, the last CTA (ticket) publishes the
// new epoch into every rank's flag slot for this rank (same protocol as exchange.cu).
DDIT_DEV void xch_signal(const EpiParams& ep) {
  if (threadIdx.x != 0 || ep.xflags[0] == nullptr) return;
  __threadfence_system();
  const unsigned int ticket = atomicAdd(ep.xcounter, 1u);
  if (ticket != gridDim.x - 1) return;
  *ep.xcounter = 0;
  __threadfence_system();
  const uint32_t e = *ep.xepoch + 1;
  *ep.xepoch = e;
  for (int q = 0; q < ep.xP; ++q)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(ep.xflags[q] + ep.xrank), "r"(e)
                 : "memory");
}

// x[r, c] += gate[b(r), c] * (acc + bias[c]) in fp32 through TMA (load, update in smem, store),
// plus an optional bf16 copy of the new x (the cross-attention query input).
// Every epilogue warp owns the 32 accumulator rows of its TMEM lane quarter and runs an
// independent pipeline over them: its residual 32x32 sub-tiles stream through a private
// RSLOTS-deep ring whose loads run RSLOTS-2 sub-tiles ahead (across tile boundaries), its own
// TMA stores leave from the same slot, and no CTA-wide barrier is involved -- the four warps
// drift freely, so one warp's HBM latency hides behind the others' math.
template <int BN, int EPI>
DDIT_DEV void epi_resid_tile(const EpiParams& ep, const CUtensorMap* tmR, const CUtensorMap* tmO2,
                             uint8_t* sE, uint64_t* rbar, uint32_t taddr, int ew, int lane,
                             int m0, int n0, const EpiCtx& cx, const ResidStream& rs,
                             int& cnt, uint32_t tempty_cl, const float* sCol) {
  constexpr int NS = BN / 32;
  constexpr bool COPY = EPI == EPI_RESID_COPY;
  static_assert(!COPY || NS % 2 == 0, "paired bf16 copy needs BN % 64 == 0");
  using Cfg = EpiCfg<BN, EPI>;
  constexpr int R = Cfg::RSLOTS;
  uint8_t* wbase = sE + ew * Cfg::WARP_BYTES;
  uint64_t* wbar = rbar + ew * R;
  const int rit = lane;  // row within the warp's slab (swizzle phase = lane & 7)
  const int row = m0 + ew * 32 + lane;
  const int grow = row < cx.M ? row : cx.M - 1;
  const float* gate_row = ep.gate ? ep.gate + (size_t)(grow / ep.rows_per_b) * ep.gate_stride : nullptr;
  const float* s_gate = sCol && ep.gate ? sCol + (size_t)(1 + grow / ep.rows_per_b) * cx.N : nullptr;
  // fused exchange: lane l copies rows 4i + l/8 (i < 8), 16 B chunk l%8 of each sub-tile row
  float* xrow[8];
  if (ep.xch) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int gr = m0 + ew * 32 + 4 * i + (lane >> 3);
      xrow[i] = gr < cx.M ? xch_row(ep, gr, ep.ldr) : nullptr;
    }
  }
#pragma unroll 1
  for (int sub = 0; sub < NS; ++sub) {
    const int slot = cnt % R;
    uint8_t* rb = wbase + slot * 4096;
    // bf16 copy buffer: per sub-tile (RESID) or per sub-tile pair (COPY; pairs never straddle a
    // tile because NS is even and cnt counts sub-tiles from 0)
    uint8_t* ob = Cfg::HAS_OB ? wbase + R * 4096 + ((COPY ? cnt >> 1 : cnt) % Cfg::NOB) * Cfg::OB : nullptr;
    const int col0 = n0 + sub * 32;
    // column vectors first: their L2 latency overlaps the waits below
    float4 bv[8], gv[8];
    if (sCol) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        bv[j] = reinterpret_cast<const float4*>(sCol + col0)[j];
        gv[j] = s_gate ? reinterpret_cast<const float4*>(s_gate + col0)[j] : make_float4(1.f, 1.f, 1.f, 1.f);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        bv[j] = ep.bias ? __ldg(reinterpret_cast<const float4*>(ep.bias + col0) + j)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        gv[j] = gate_row ? __ldg(reinterpret_cast<const float4*>(gate_row + col0) + j)
                         : make_float4(1.f, 1.f, 1.f, 1.f);
      }
    }
    if (lane == 0) {
      // this warp's stores up to sub-tile cnt-1-(NOB-2) have read their smem, so the ring slot
      // of sub-tile cnt+RAHEAD and the next bf16 buffer are free again
      constexpr int AH = Cfg::RAHEAD;
      bulk_wait_read<Cfg::NOB - 2>();
      if (ew == 0) EPI_TRACE(384 + 16 * (cnt / NS) + sub);
      resid_issue<R>(rs, NS, cnt + AH, ew * 32, tmR, wbase, wbar);
    }
    if (ew == 0 && lane == 0) EPI_TRACE(256 + 16 * (cnt / NS) + 2 * sub);
    mbar_wait(&wbar[slot], (cnt / R) & 1);
    if (ew == 0 && lane == 0) EPI_TRACE(256 + 16 * (cnt / NS) + 2 * sub + 1);
    uint32_t r[32];
    tmem_ld_x32(taddr + sub * 32, r);
    tmem_ld_wait();
    if (ew == 0 && lane == 0) EPI_TRACE(512 + 16 * (cnt / NS) + sub);
    if (sub == NS - 1) {
      // lane 31 arrives: its release has no outstanding TMA issue / global traffic to order
      // (lane 0 issues the warp's bulk copies), so it does not stall the warp
      tc_fence_before();
      __syncwarp();
      if (lane == 31) mbar_arrive_cl_relaxed(tempty_cl);
    }
    const uint32_t rbase = smem_u32(rb);
    float nv[32];
    float4 xv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) xv[j] = ld_shared_f4(rbase + sw128(rit, j));  // all loads in flight
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 b = bv[j], g = gv[j], x = xv[j];
      // x + (g * (acc + b)) rounded step by step (no FMA contraction): the reduce-add epilogue
      // (EPI_RESID_RED) computes exactly this, so DoP-P ranks that exchange stay bit-exact
      nv[4 * j + 0] = __fadd_rn(x.x, __fmul_rn(g.x, __fadd_rn(__uint_as_float(r[4 * j + 0]), b.x)));
      nv[4 * j + 1] = __fadd_rn(x.y, __fmul_rn(g.y, __fadd_rn(__uint_as_float(r[4 * j + 1]), b.y)));
      nv[4 * j + 2] = __fadd_rn(x.z, __fmul_rn(g.z, __fadd_rn(__uint_as_float(r[4 * j + 2]), b.z)));
      nv[4 * j + 3] = __fadd_rn(x.w, __fmul_rn(g.w, __fadd_rn(__uint_as_float(r[4 * j + 3]), b.w)));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      st_shared_v4(rbase + sw128(rit, j), __float_as_uint(nv[4 * j]), __float_as_uint(nv[4 * j + 1]),
                   __float_as_uint(nv[4 * j + 2]), __float_as_uint(nv[4 * j + 3]));
    if (COPY) {  // chunks 4h..4h+3 of the pair's 128 B row, h = sub-tile parity
      const uint32_t obase = smem_u32(ob);
      const int h = cnt & 1;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        st_shared_v4(obase + sw128(rit, 4 * h + j), pack_bf16(nv[8 * j], nv[8 * j + 1]),
                     pack_bf16(nv[8 * j + 2], nv[8 * j + 3]), pack_bf16(nv[8 * j + 4], nv[8 * j + 5]),
                     pack_bf16(nv[8 * j + 6], nv[8 * j + 7]));
    } else if (Cfg::HAS_OB && ep.out2) {
      const uint32_t obase = smem_u32(ob);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        st_shared_v4(obase + sw64(rit, j), pack_bf16(nv[8 * j], nv[8 * j + 1]),
                     pack_bf16(nv[8 * j + 2], nv[8 * j + 3]), pack_bf16(nv[8 * j + 4], nv[8 * j + 5]),
                     pack_bf16(nv[8 * j + 6], nv[8 * j + 7]));
    }
    if (ew == 0 && lane == 0) EPI_TRACE(768 + 16 * (cnt / NS) + sub);
    if (ep.xch) {  // rows go to their owner rank (peer stores), 4 whole 128 B rows per instruction
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (xrow[i] != nullptr) {
          const float4 v = ld_shared_f4(rbase + sw128(4 * i + (lane >> 3), lane & 7));
          *reinterpret_cast<float4*>(xrow[i] + col0 + 4 * (lane & 7)) = v;
        }
      }
      fence_async_smem();  // generic reads of the slot before its next TMA load
      __syncwarp();
    } else {
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmR, rb, col0, m0 + ew * 32);
        if (COPY) {
          if (cnt & 1) tma_store_2d(tmO2, ob, col0 - 32, m0 + ew * 32);
        } else if (Cfg::HAS_OB && ep.out2) {
          tma_store_2d(tmO2, ob, col0, m0 + ew * 32);
        }
        bulk_commit();
      }
    }
    if (ew == 0 && lane == 0) EPI_TRACE(640 + 16 * (cnt / NS) + sub);
    ++cnt;
  }
}

DDIT_DEV void tma_reduce_add_2d(const void* tmap, const void* smem_src, int c0, int c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
      : "memory");
}

// x[r, c] += gate[b(r), c] * (acc + bias[c]) without reading x: every warp stages y = gate *
// (acc + bias) for its 32 rows x 32 columns in a ring of RSLOTS swizzled fp32 buffers and sends
// it to x with a TMA reduce-add (the L2 computes x + y, round-to-nearest -- the same two
// roundings as the load / update / store path, which keeps DoP-P bit-exact). The only wait is for
// a buffer's previous reduce to finish reading shared memory, RSLOTS - 1 sub-tiles later.
template <int BN>
DDIT_DEV void epi_red_tile(const EpiParams& ep, const CUtensorMap* tmR, uint8_t* sE,
                           uint32_t taddr, int ew, int lane, int m0, int n0, const EpiCtx& cx,
                           int& cnt, uint32_t tempty_cl, const float* sCol) {
  constexpr int NS = BN / 32;
  using Cfg = EpiCfg<BN, EPI_RESID_RED>;
  constexpr int R = Cfg::RSLOTS;
  uint8_t* wbase = sE + ew * Cfg::WARP_BYTES;
  const int row = m0 + ew * 32 + lane;
  const int grow = row < cx.M ? row : cx.M - 1;
  const float* gate_row = ep.gate ? ep.gate + (size_t)(grow / ep.rows_per_b) * ep.gate_stride : nullptr;
  const float* s_gate = sCol && ep.gate ? sCol + (size_t)(1 + grow / ep.rows_per_b) * cx.N : nullptr;
#pragma unroll 1
  for (int sub = 0; sub < NS; ++sub) {
    uint8_t* rb = wbase + (cnt % R) * 4096;
    const int col0 = n0 + sub * 32;
    float4 bv[8], gv[8];
    if (sCol) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        bv[j] = reinterpret_cast<const float4*>(sCol + col0)[j];
        gv[j] = s_gate ? reinterpret_cast<const float4*>(s_gate + col0)[j] : make_float4(1.f, 1.f, 1.f, 1.f);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        bv[j] = ep.bias ? __ldg(reinterpret_cast<const float4*>(ep.bias + col0) + j)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        gv[j] = gate_row ? __ldg(reinterpret_cast<const float4*>(gate_row + col0) + j)
                         : make_float4(1.f, 1.f, 1.f, 1.f);
      }
    }
    uint32_t r[32];
    tmem_ld_x32(taddr + sub * 32, r);
    if (lane == 0) bulk_wait_read<R - 1>();  // the reduce that last used this buffer has read it
    tmem_ld_wait();
    if (sub == NS - 1) {
      tc_fence_before();
      __syncwarp();
      if (lane == 31) mbar_arrive_cl_relaxed(tempty_cl);
    }
    __syncwarp();
    const uint32_t rbase = smem_u32(rb);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 b = bv[j], g = gv[j];
      st_shared_v4(rbase + sw128(lane, j),
                   __float_as_uint(__fmul_rn(g.x, __fadd_rn(__uint_as_float(r[4 * j + 0]), b.x))),
                   __float_as_uint(__fmul_rn(g.y, __fadd_rn(__uint_as_float(r[4 * j + 1]), b.y))),
                   __float_as_uint(__fmul_rn(g.z, __fadd_rn(__uint_as_float(r[4 * j + 2]), b.z))),
                   __float_as_uint(__fmul_rn(g.w, __fadd_rn(__uint_as_float(r[4 * j + 3]), b.w))));
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_reduce_add_2d(tmR, rb, col0, m0 + ew * 32);
      bulk_commit();
    }
    ++cnt;
  }
}

// ------------------------------------------------------------------ epilogue: QKV
// The 144-column tile holds two whole heads (head_dim 72) of one of q/k/v.
// q,k: bias -> per-head RMSNorm (weight) -> optional interleaved RoPE by frame index.
// NH heads per tile in HS-column slots: HS = 72 (the QKV matrix as is, BN 144) or HS = 80 (the
// weight rows padded per head with 8 zero rows, BN 240 = 3 heads: the shared-memory-cheaper
// tile shape, §3 of DESIGN.md); the output always has 72-column head slots. The padded columns
// are computed (zero) and dropped.
template <int NH, int HS>
DDIT_DEV void epi_qkv_tile(const EpiParams& ep, const CUtensorMap* tmO, uint8_t* sE,
                           uint32_t taddr, int rit, int m0, int n0, bool elected, int& cnt,
                           uint32_t tempty_cl, int lane, const float* sCol) {
  constexpr int HD = 72;
  const int heads = ep.hidden / HD;
  const int row = m0 + rit;
  const int pos = ep.rope ? (row / ep.rope_S) % ep.rope_T : 0;
  // per-warp staging (32 rows x 144 B, double-buffered) and per-warp TMA stores: the four
  // epilogue warps never wait for each other
  const int ew = rit >> 5;
#pragma unroll 1
  for (int h = 0; h < NH; ++h) {
    const int hi = n0 / HS + h;        // head slot in [0, 3 heads)
    const int section = hi / heads;    // 0 q, 1 k, 2 v
    uint8_t* sb = sE + ew * 9216 + (cnt & 1) * 4608;
    const uint32_t sbase = smem_u32(sb) + lane * 144;
    if (lane == 0) bulk_wait_read<1>();  // this warp's store of two heads ago has read sb
    __syncwarp();
    uint32_t r[72];
    tmem_ld_x32(taddr + h * HS, r);
    tmem_ld_x32(taddr + h * HS + 32, r + 32);
    tmem_ld_32x32b_x8(taddr + h * HS + 64, r + 64);
    tmem_ld_wait();
    if (h == NH - 1) {
      tc_fence_before();
      __syncwarp();
      if (lane == 31) mbar_arrive_cl_relaxed(tempty_cl);
    }
    const int c0 = n0 + h * HS;  // bias column (same slot layout as the GEMM's N)
    float v[72];
    float ss = 0.f;
#pragma unroll
    for (int q = 0; q < 18; ++q) {
      const float4 b = sCol ? reinterpret_cast<const float4*>(sCol + c0)[q]
                            : __ldg(reinterpret_cast<const float4*>(ep.bias + c0) + q);
      v[4 * q + 0] = __uint_as_float(r[4 * q + 0]) + b.x;
      v[4 * q + 1] = __uint_as_float(r[4 * q + 1]) + b.y;
      v[4 * q + 2] = __uint_as_float(r[4 * q + 2]) + b.z;
      v[4 * q + 3] = __uint_as_float(r[4 * q + 3]) + b.w;
      ss += v[4 * q] * v[4 * q] + v[4 * q + 1] * v[4 * q + 1] + v[4 * q + 2] * v[4 * q + 2] +
            v[4 * q + 3] * v[4 * q + 3];
    }
    if (section < 2) {
      const float inv = rsqrtf(ss * (1.0f / HD) + ep.eps);
      const float* w = section == 0 ? ep.qnorm_w : ep.knorm_w;
#pragma unroll
      for (int q = 0; q < 18; ++q) {
        const float4 wq = __ldg(reinterpret_cast<const float4*>(w) + q);
        v[4 * q + 0] *= inv * wq.x;
        v[4 * q + 1] *= inv * wq.y;
        v[4 * q + 2] *= inv * wq.z;
        v[4 * q + 3] *= inv * wq.w;
      }
      if (ep.rope) {
        const float4* tab = reinterpret_cast<const float4*>(ep.rope_tab + pos * (HD / 2));
#pragma unroll
        for (int q = 0; q < 18; ++q) {  // pairs (4q, 4q+1), (4q+2, 4q+3)
          const float4 cs = __ldg(tab + q);
          const float a0 = v[4 * q], a1 = v[4 * q + 1], a2 = v[4 * q + 2], a3 = v[4 * q + 3];
          v[4 * q + 0] = a0 * cs.x - a1 * cs.y;
          v[4 * q + 1] = a1 * cs.x + a0 * cs.y;
          v[4 * q + 2] = a2 * cs.z - a3 * cs.w;
          v[4 * q + 3] = a3 * cs.z + a2 * cs.w;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 9; ++j)
      st_shared_v4(sbase + j * 16, pack_bf16(v[8 * j], v[8 * j + 1]),
                   pack_bf16(v[8 * j + 2], v[8 * j + 3]), pack_bf16(v[8 * j + 4], v[8 * j + 5]),
                   pack_bf16(v[8 * j + 6], v[8 * j + 7]));
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tmO, sb, hi * HD, m0 + ew * 32);
      bulk_commit();
    }
    ++cnt;
  }
}

// ------------------------------------------------------------------ kernel
template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmO,
                        const __grid_constant__ CUtensorMap tmR,
                        const __grid_constant__ CUtensorMap tmO2, int M, int N, int K,
                        const __grid_constant__ EpiParams ep) {
  using Cfg = GemmCfg<BN, EPI>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sE = smem + STAGES * Cfg::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sE + EpiCfg<BN, EPI>::BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + kRBars);

  const int warp = warp_id();
  const int lane = lane_id();
  EpiCtx cx;
  cx.M = M;
  cx.N = N;
  cx.m_tiles = (M + BM - 1) / BM;
  cx.n_tiles = N / BN;
  cx.num_tiles = cx.m_tiles * cx.n_tiles;
  const int n_tiles = cx.n_tiles;
  const int num_tiles = cx.num_tiles;
  const int k_blocks = (K + BK - 1) / BK;  // TMA zero-fills the K tail

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmO);
    if constexpr (is_resid(EPI)) tma_prefetch_desc(&tmR);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    for (int i = 0; i < kRBars; ++i) mbar_init(&rbar[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_a = l2_policy_evict_first();
      const uint64_t pol_b = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m_blk = tile / n_tiles;
        const int n_blk = tile % n_tiles;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          tma_load_2d_hint(sA + stage * Cfg::A_BYTES, &tmA, &full[stage], kb * BK, m_blk * BM, pol_a);
          tma_load_2d_hint(sB + stage * Cfg::B_BYTES, &tmB, &full[stage], kb * BK, n_blk * BN, pol_b);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      pdl_trigger();  // all loads issued: dependents may start their prologue
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_bf16(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * kAccStride;
      for (int kb = 0; kb < k_blocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_base = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            umma_bf16_ss(d_tmem, make_sdesc_sw128(a_base + k * 32), make_sdesc_sw128(b_base + k * 32),
                         idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (kb == k_blocks - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int rit = ew * 32 + lane;  // row within the tile
    const bool elected = (ew == 0 && lane == 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    int cnt = 0;
    const ResidStream rs{(int)blockIdx.x, (int)gridDim.x, num_tiles, n_tiles, BM, 0};
    const float* sCol = nullptr;
    if constexpr (!is_resid(EPI) && EpiCfg<BN, EPI>::COL_BYTES > 0)
      sCol = epi_stage_cols<EpiCfg<BN, EPI>::COL_BYTES>(
          ep, reinterpret_cast<float*>(sE + 2 * EpiCfg<BN, EPI>::BUF), M, N, ew * 32 + lane);
    if constexpr (is_resid(EPI)) {
      constexpr int R = EpiCfg<BN, EPI>::RSLOTS;
      sCol = epi_stage_cols<EpiCfg<BN, EPI>::COL_BYTES>(
          ep, reinterpret_cast<float*>(sE + 4 * EpiCfg<BN, EPI>::WARP_BYTES), M, N, ew * 32 + lane);
      if (elected) {  // residual tiles 0 and 1 into L2
        resid_prefetch_l2<BN>(rs, 0, &tmO);
        resid_prefetch_l2<BN>(rs, 1, &tmO);
      }
      if (EPI != EPI_RESID_RED && lane == 0)  // the first R-2 residual sub-tiles of this warp's slab
        for (int j = 0; j < EpiCfg<BN, EPI>::RAHEAD; ++j)
          resid_issue<R>(rs, BN / 32, j, ew * 32, &tmR, sE + ew * EpiCfg<BN, EPI>::WARP_BYTES, rbar + ew * R);
    }
    int tix = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m0 = (tile / n_tiles) * BM;
      const int n0 = (tile % n_tiles) * BN;
      if constexpr (is_resid(EPI)) {  // two tiles ahead: lands in L2 well before its epilogue
        if (elected) resid_prefetch_l2<BN>(rs, tix + 2, &tmO);
        ++tix;
      }
      if (ew == 0 && lane == 0) EPI_TRACE(128 + 2 * (tix - 1));
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (ew == 0 && lane == 0) EPI_TRACE(128 + 2 * (tix - 1) + 1);
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * kAccStride;
      const uint32_t tcl = cluster_addr(&tempty[acc], 0);
      if constexpr (EPI == EPI_QKV) {
        epi_qkv_tile<BN == 240 ? 3 : 2, BN == 240 ? 80 : 72>(ep, &tmO, sE, taddr, rit, m0, n0, elected, cnt, tcl, lane, sCol);
      } else if constexpr (EPI == EPI_RESID_RED) {
        epi_red_tile<BN>(ep, &tmR, sE, taddr, ew, lane, m0, n0, cx, cnt, tcl, sCol);
      } else if constexpr (is_resid(EPI)) {
        epi_resid_tile<BN, EPI>(ep, &tmR, &tmO2, sE, rbar, taddr, ew, lane, m0, n0, cx, rs, cnt, tcl, sCol);
      } else {
        epi_plain_tile<BN, EPI>(ep, &tmO, sE, taddr, rit, m0, n0, elected, cnt, tcl, lane, sCol);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (elected || ((is_resid(EPI) || EPI == EPI_QKV) && lane == 0)) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (is_resid(EPI)) {
    if (ep.xch) xch_signal(ep);
  }
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------ 2-CTA kernel
// cta_group::2: a cluster of two CTAs (one TPC) computes a 256 x BN tile. CTA r holds rows
// [128r, 128r+128) of A and rows [r*BN/2, (r+1)*BN/2) of B in its smem and the accumulator rows
// [128r, 128r+128) x BN in its TMEM; the leader (rank 0) issues tcgen05.mma.cta_group::2 with
// M = 256. Each SM streams half the B operand of the 1-CTA kernel.
template <int BN, int EPI, int WIDE = 1>
struct GemmCfg2 {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = WIDE * (BN / 2) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_BYTES = 512;
  static constexpr int BUDGET = 232448 - 1024 - BAR_BYTES - EpiCfg<BN, EPI>::BYTES;
  static constexpr int STAGES_RAW = BUDGET / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 10 ? 10 : STAGES_RAW;
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + EpiCfg<BN, EPI>::BYTES + BAR_BYTES;
  static_assert(B_BYTES % 1024 == 0, "B half-tile must keep 1024 B swizzle-atom alignment");
  static_assert(BN % 16 == 0 && (BN / 2) % 8 == 0 && BN <= 256, "invalid UMMA N for cta_group::2");
  static_assert(STAGES >= 3, "pipeline too shallow");
};

// WIDE = 2: each tile is 256 x 2BN, computed as two N = BN MMAs per k-step into the two TMEM
// accumulator halves [0, BN) and [BN, 2BN) (one tile in flight, no double buffer): per k-block the
// A stage is written once for 2BN output columns, which lowers the shared-memory traffic per
// FLOP; the epilogue drains half 0 then half 1, each with the BN epilogue.
template <int BN, int EPI, int WIDE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2_bf16_tn_kernel(const __grid_constant__ CUtensorMap tmA,
                         const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmO,
                         const __grid_constant__ CUtensorMap tmR,
                         const __grid_constant__ CUtensorMap tmO2, int M, int N, int K,
                         const __grid_constant__ EpiParams ep) {
  using Cfg = GemmCfg2<BN, EPI, WIDE>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int BM2 = 2 * BM;
  constexpr int TW = WIDE * BN;  // output columns per tile
  static_assert(WIDE == 1 || TW <= 512, "wide tile exceeds TMEM");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sE = smem + STAGES * Cfg::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sE + EpiCfg<BN, EPI>::BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + kRBars);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_rank();
  const int cid = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  EpiCtx cx;
  cx.M = M;
  cx.N = N;
  cx.m_tiles = (M + BM2 - 1) / BM2;
  cx.n_tiles = N / TW;
  cx.num_tiles = cx.m_tiles * cx.n_tiles;
  const int n_tiles = cx.n_tiles;
  const int num_tiles = cx.num_tiles;
  const int k_blocks = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmO);
    if constexpr (is_resid(EPI)) tma_prefetch_desc(&tmR);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    for (int i = 0; i < kRBars; ++i) mbar_init(&rbar[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  __syncthreads();  // (a CTA barrier is implied; explicit for compute-sanitizer racecheck)
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();

  if (warp == 0) {
    if (elect_one()) {  // ---- producer (both CTAs): own halves of A and B -> leader's barrier
      const uint64_t pol_a = l2_policy_evict_first();
      const uint64_t pol_b = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cid; tile < num_tiles; tile += nclusters) {
        const int m0 = (tile / n_tiles) * BM2 + rank * BM;
        const int nb0 = (tile % n_tiles) * TW + rank * (BN / 2);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
          const uint32_t bar0 = cluster_addr(&full[stage], 0);
          tma_load_2d_cg2(sA + stage * Cfg::A_BYTES, &tmA, bar0, kb * BK, m0, pol_a);
#pragma unroll
          for (int h = 0; h < WIDE; ++h)  // half h: output columns [h BN, h BN + BN) of the tile
            tma_load_2d_cg2(sB + stage * Cfg::B_BYTES + h * (BN / 2) * BK * 2, &tmB, bar0, kb * BK,
                            nb0 + h * BN, pol_b);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      pdl_trigger();
    }
  } else if (warp == 1) {
    if (rank == 0) {  // ---- MMA issuer (leader CTA only)
      constexpr uint32_t idesc = make_idesc_bf16(BM2, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int tt = 0;
      for (int tile = cid; tile < num_tiles; tile += nclusters, ++tt) {
        if (lane == 0) EPI_TRACE(2 * tt);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        if constexpr (WIDE == 2) mbar_wait(&tempty[1], acc_phase ^ 1);  // both halves drained
        tc_fence_after();
        if (lane == 0) EPI_TRACE(2 * tt + 1);
        const uint32_t d_tmem = tmem_base + (WIDE == 2 ? 0u : acc * kAccStride);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0 && kb == 0) EPI_TRACE(64 + 2 * tt);
          if (lane == 0 && kb == k_blocks - 1) EPI_TRACE(64 + 2 * tt + 1);
          if (elect_one()) {
            const uint32_t a_base = smem_u32(sA + stage * Cfg::A_BYTES);
            const uint32_t b_base = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
#pragma unroll
              for (int h = 0; h < WIDE; ++h)
                umma_bf16_ss_cg2(d_tmem + h * BN, make_sdesc_sw128(a_base + k * 32),
                                 make_sdesc_sw128(b_base + h * (BN / 2) * BK * 2 + k * 32), idesc,
                                 (kb | k) != 0);
            umma_commit_cg2_mc(&empty[stage]);
            if (kb == k_blocks - 1) {
              umma_commit_cg2_mc(&tfull[acc]);
              if constexpr (WIDE == 2) umma_commit_cg2_mc(&tfull[1]);
            }
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (WIDE == 2) {
          acc_phase ^= 1;
        } else {
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {  // ---- epilogue (both CTAs): own 128 accumulator rows
    const int ew = warp - 4;
    const int rit = ew * 32 + lane;
    const bool elected = (ew == 0 && lane == 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    int cnt = 0;
    const ResidStream rs{cid, nclusters, num_tiles, n_tiles, BM2, (int)rank * BM};
    const float* sCol = nullptr;
    if constexpr (!is_resid(EPI) && EpiCfg<BN, EPI>::COL_BYTES > 0)
      sCol = epi_stage_cols<EpiCfg<BN, EPI>::COL_BYTES>(
          ep, reinterpret_cast<float*>(sE + 2 * EpiCfg<BN, EPI>::BUF), M, N, ew * 32 + lane);
    if constexpr (is_resid(EPI)) {
      constexpr int R = EpiCfg<BN, EPI>::RSLOTS;
      sCol = epi_stage_cols<EpiCfg<BN, EPI>::COL_BYTES>(
          ep, reinterpret_cast<float*>(sE + 4 * EpiCfg<BN, EPI>::WARP_BYTES), M, N, ew * 32 + lane);
      if (elected) {  // residual tiles 0 and 1 into L2
        resid_prefetch_l2<BN>(rs, 0, &tmO);
        resid_prefetch_l2<BN>(rs, 1, &tmO);
      }
      if (EPI != EPI_RESID_RED && lane == 0)  // the first R-2 residual sub-tiles of this warp's slab
        for (int j = 0; j < EpiCfg<BN, EPI>::RAHEAD; ++j)
          resid_issue<R>(rs, BN / 32, j, ew * 32, &tmR, sE + ew * EpiCfg<BN, EPI>::WARP_BYTES, rbar + ew * R);
    }
    int tix = 0;
    for (int tile = cid; tile < num_tiles; tile += nclusters) {
      const int m0 = (tile / n_tiles) * BM2 + rank * BM;
      const int nt0 = (tile % n_tiles) * TW;
      if constexpr (is_resid(EPI)) {  // two tiles ahead: lands in L2 well before its epilogue
        if (elected) {
          if constexpr (WIDE == 2) {
            resid_prefetch_l2_wide<BN>(rs, tix + 2, &tmO);
          } else {
            resid_prefetch_l2<BN>(rs, tix + 2, &tmO);
          }
        }
        ++tix;
      }
#pragma unroll 1
      for (int h = 0; h < WIDE; ++h) {
        const int hb = WIDE == 2 ? h : acc;  // accumulator half / buffer
        const int n0 = nt0 + h * BN;
        if (ew == 0 && lane == 0) EPI_TRACE(128 + 2 * (tix - 1));
        mbar_wait(&tfull[hb], acc_phase);
        tc_fence_after();
        if (ew == 0 && lane == 0) EPI_TRACE(128 + 2 * (tix - 1) + 1);
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) +
                               (WIDE == 2 ? hb * BN : hb * kAccStride);
        const uint32_t tcl = cluster_addr(&tempty[hb], 0);
        if constexpr (EPI == EPI_QKV) {
          epi_qkv_tile<BN == 240 ? 3 : 2, BN == 240 ? 80 : 72>(ep, &tmO, sE, taddr, rit, m0, n0, elected, cnt, tcl, lane, sCol);
        } else if constexpr (EPI == EPI_RESID_RED) {
          epi_red_tile<BN>(ep, &tmR, sE, taddr, ew, lane, m0, n0, cx, cnt, tcl, sCol);
        } else if constexpr (is_resid(EPI)) {
          epi_resid_tile<BN, EPI>(ep, &tmR, &tmO2, sE, rbar, taddr, ew, lane, m0, n0, cx, rs, cnt, tcl, sCol);
        } else {
          epi_plain_tile<BN, EPI>(ep, &tmO, sE, taddr, rit, m0, n0, elected, cnt, tcl, lane, sCol);
        }
      }
      if constexpr (WIDE == 2) {
        acc_phase ^= 1;
      } else {
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
    if (elected || ((is_resid(EPI) || EPI == EPI_QKV) && lane == 0)) bulk_wait<0>();
  }
  tc_fence_before();
  cluster_sync_all();
  if constexpr (is_resid(EPI)) {
    if (ep.xch) xch_signal(ep);
  }
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(kTmemCols)
                 : "memory");
  }
}

// ------------------------------------------------------------------ host
static thread_local char g_err[512];
const char* gemm_last_error() { return g_err; }

typedef CUresult (*PFN_tmapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                        const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                        const cuuint32_t*, CUtensorMapInterleave,
                                        CUtensorMapSwizzle, CUtensorMapL2promotion,
                                        CUtensorMapFloatOOBfill);

static PFN_tmapEncodeTiled get_encode() {
  static PFN_tmapEncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_tmapEncodeTiled>(p);
  });
  return fn;
}

// 2-D tensor map over a row-major [rows, cols] matrix (row stride ld elements) with box
// [box_rows, box_cols]; zero fill out of bounds on loads, clipping on stores.
static int make_tmap(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int esize, int rows,
                     int cols, int ld, int box_rows, int box_cols, CUtensorMapSwizzle sw) {
  PFN_tmapEncodeTiled enc = get_encode();
  if (!enc) {
    snprintf(g_err, sizeof g_err, "cuTensorMapEncodeTiled unavailable");
    return -1;
  }
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)ld * esize};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_err, sizeof g_err,
             "cuTensorMapEncodeTiled failed (%d) rows=%d cols=%d ld=%d box=%dx%d", (int)r, rows,
             cols, ld, box_rows, box_cols);
    return -1;
  }
  return 0;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static bool bn_ok(int bn, int epi) {
  if (epi == EPI_QKV) return bn == 144 || bn == 240;
  if (epi == EPI_RESID_COPY) return bn == 128 || bn == 192 || bn == 256;
  if (bn == 0) return false;
  return bn == 96 || bn == 128 || bn == 192 || bn == 256;
}

int gemm_plan_init(GemmPlan* p, const void* A, int lda, const void* B, int ldb, int M, int N,
                   int K, int epi, const EpiParams& ep, int bn) {
  return gemm_plan_init_cta(p, A, lda, B, ldb, M, N, K, epi, ep, bn, two_cta_enabled() ? 1 : 0);
}

// Tile choice for an M x N output on this GPU: fewest "tile-waves" weighted by the per-tile
// efficiency measured at large M (240p, K = 1152) -- 2-CTA 256 x BN tiles over #SMs/2 pairs,
// 1-CTA 128 x BN tiles over #SMs. Only M/N tiling changes (never the K order), so every choice
// gives bit-identical results: a DoP-P rank with a small M may pick a different tile than DoP 1.
void gemm_pick_tile(int M, int N, int epi, int* bn_out, int* two_out) {
  struct Cand { int bn, two; double eff; };
  static const Cand cands[] = {{256, 1, 1.0}, {192, 1, 1.0},  {144, 1, 1.0},  {128, 1, 0.90},
                               {96, 1, 0.72}, {256, 0, 0.85}, {192, 0, 0.85}, {144, 0, 0.85},
                               {128, 0, 0.74}, {96, 0, 0.62}};
  const int sms = num_sms();
  double best = 1e30;
  int bbn = 0, btwo = 0;
  for (const Cand& c : cands) {
    if (c.two && !two_cta_enabled()) continue;
    if ((epi == EPI_QKV) != (c.bn == 144) || N % c.bn) continue;
    const int bm = c.two ? 2 * BM : BM, units = c.two ? sms / 2 : sms;
    const long tiles = (long)((M + bm - 1) / bm) * (N / c.bn);
    const double cost = (double)((tiles + units - 1) / units) * c.bn / c.eff;
    if (cost < best - 1e-9) {
      best = cost;
      bbn = c.bn;
      btwo = c.two;
    }
  }
  *bn_out = bbn;
  *two_out = btwo;
}

int gemm_plan_init_cta(GemmPlan* p, const void* A, int lda, const void* B, int ldb, int M, int N,
                       int K, int epi, const EpiParams& ep, int bn, int two_cta) {
  if (!bn_ok(bn, epi)) {
    snprintf(g_err, sizeof g_err, "unsupported BN %d for epilogue %d", bn, epi);
    return -2;
  }
  if (M <= 0 || N % bn != 0 || K <= 0) {
    snprintf(g_err, sizeof g_err, "bad GEMM shape M=%d N=%d K=%d BN=%d", M, N, K, bn);
    return -2;
  }
  if (epi == EPI_QKV && (ep.hidden % 144 != 0 || N != (bn == 240 ? 3 * ep.hidden / 72 * 80 : 3 * ep.hidden))) {
    snprintf(g_err, sizeof g_err, "EPI_QKV needs hidden %% 144 == 0 and N = 3 heads x (72 | 80 at BN 240)");
    return -2;
  }
  if ((lda * 2) % 16 || (ldb * 2) % 16 || (reinterpret_cast<uintptr_t>(A) & 15) ||
      (reinterpret_cast<uintptr_t>(B) & 15)) {
    snprintf(g_err, sizeof g_err, "GEMM operands must be 16-byte aligned");
    return -2;
  }
  memset(p, 0, sizeof *p);
  p->two_cta = two_cta ? 1 : 0;
  const auto BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const auto F32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  if (make_tmap(&p->tmA, A, BF, 2, M, K, lda, BM, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return -3;
  const int bbox = p->two_cta ? bn / 2 : bn;
  if (make_tmap(&p->tmB, B, BF, 2, N, K, ldb, bbox, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return -3;
  switch (epi) {
    case EPI_BF16:
    case EPI_GELU_BF16: {
      const bool wide = bn % 64 == 0;
      if (!ep.out || make_tmap(&p->tmO, ep.out, BF, 2, M, N, ep.ldo, BM, wide ? 64 : 32,
                               wide ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B))
        return -3;
      break;
    }
    case EPI_F32:
      if (!ep.out || make_tmap(&p->tmO, ep.out, F32, 4, M, N, ep.ldo, BM, 32, CU_TENSOR_MAP_SWIZZLE_128B))
        return -3;
      break;
    case EPI_QKV:  // output: 72-column head slots whatever the GEMM's slot width
      if (!ep.out || make_tmap(&p->tmO, ep.out, BF, 2, M, 3 * ep.hidden, ep.ldo, 32, 72, CU_TENSOR_MAP_SWIZZLE_NONE))
        return -3;
      break;
    case EPI_RESID:
    case EPI_RESID_COPY:
    case EPI_RESID_RED:
      // with a bf16 copy and BN % 64 == 0, the copy leaves in 64-column boxes (EPI_RESID_COPY);
      // without copy or exchange the update is a TMA reduce-add (EPI_RESID_RED)
      if (ep.out2 && bn % 64 == 0) epi = EPI_RESID_COPY;
      if (!ep.out2 && !ep.xch && resid_red_enabled()) epi = EPI_RESID_RED;
      if (epi == EPI_RESID_RED && (ep.out2 || ep.xch)) epi = EPI_RESID;
      if (epi == EPI_RESID_COPY && (!ep.out2 || bn % 64)) {
        snprintf(g_err, sizeof g_err, "EPI_RESID_COPY needs out2 and BN %% 64 == 0");
        return -2;
      }
      if (!ep.resid ||
          make_tmap(&p->tmR, ep.resid, F32, 4, M, N, ep.ldr, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))
        return -3;
      if (epi == EPI_RESID_COPY
              ? make_tmap(&p->tmO2, ep.out2, BF, 2, M, N, ep.ldo2, 32, 64, CU_TENSOR_MAP_SWIZZLE_128B)
              : ep.out2 && make_tmap(&p->tmO2, ep.out2, BF, 2, M, N, ep.ldo2, 32, 32,
                                     CU_TENSOR_MAP_SWIZZLE_64B))
        return -3;
      // tmO (unused by this epilogue) carries the whole-tile map for the L2 prefetch
      if (make_tmap(&p->tmO, ep.resid, F32, 4, M, N, ep.ldr, BM, bn, CU_TENSOR_MAP_SWIZZLE_NONE))
        return -3;
      if (!ep.out2) p->tmO2 = p->tmR;
      break;
    default:
      snprintf(g_err, sizeof g_err, "unknown epilogue %d", epi);
      return -2;
  }
  p->M = M;
  p->N = N;
  p->K = K;
  p->bn = bn;
  p->epi = epi;
  p->ep = ep;
  // 256 x 384 tiles only where the long K loop hides the un-overlapped epilogue (fc2, K = 4608:
  // 94.0 -> 91.3 us; at K = 1152 they lose 13-16 %, scripts/wide_probe.py); bit-identical results
  gemm_plan_refresh(p);
  return 0;
}

// Tile shape and launch grid from the plan's current epilogue parameters (an exchange attached
// after the plan was built turns the reduce-add into load / update / store, which has no wide
// tile): called at plan build and by the runtime after it edits a plan's EpiParams.
void gemm_plan_refresh(GemmPlan* p) {
  if (p->bn <= 0 || p->M <= 0) return;  // never built (a rank without rows in this layout)
  const int M = p->M, N = p->N, K = p->K, bn = p->bn, epi = p->epi;
  const bool red = epi == EPI_RESID_RED && !p->ep.xch && !p->ep.out2;
  p->wide = p->two_cta && bn == 192 && N % (2 * bn) == 0 && K >= 4096 && gemm_wide_enabled() &&
            (red || epi == EPI_BF16) && !p->ep.xch;
  if (p->two_cta) {
    const int tiles = ((M + 2 * BM - 1) / (2 * BM)) * (N / (bn * (p->wide ? 2 : 1)));
    const int clusters = num_sms() / 2;
    p->grid = 2 * (tiles < clusters ? tiles : clusters);
  } else {
    const int tiles = ((M + BM - 1) / BM) * (N / bn);
    p->grid = tiles < num_sms() ? tiles : num_sms();
  }
}

static int g_resid_red = -1;
bool resid_red_enabled() {
  if (g_resid_red < 0) {
    const char* e = getenv("DDIT_RESID_RED");
    g_resid_red = (e && e[0] == '0') ? 0 : 1;
  }
  return g_resid_red != 0;
}
void set_resid_red(int on) { g_resid_red = on ? 1 : 0; }

static int g_pdl = -1;
bool pdl_enabled() {
  if (g_pdl < 0) {
    const char* e = getenv("DDIT_PDL");
    g_pdl = (e && e[0] == '0') ? 0 : 1;
  }
  return g_pdl != 0;
}
void set_pdl(int on) { g_pdl = on ? 1 : 0; }

static int g_wide = -1;
bool gemm_wide_enabled() {
  if (g_wide < 0) {
    const char* e = getenv("DDIT_GEMM_WIDE");
    g_wide = (e && e[0] == '0') ? 0 : 1;
  }
  return g_wide != 0;
}
void set_gemm_wide(int on) { g_wide = on ? 1 : 0; }

static int g_two_cta = -1;
bool two_cta_enabled() {
  if (g_two_cta < 0) {
    const char* e = getenv("DDIT_GEMM_2CTA");
    g_two_cta = (e && e[0] == '0') ? 0 : 1;
  }
  return g_two_cta != 0;
}
void set_two_cta(int on) { g_two_cta = on ? 1 : 0; }

template <int BN, int EPI, int WIDE>
static int launch_t2w(const GemmPlan* p, cudaStream_t s) {
  constexpr int smem = GemmCfg2<BN, EPI, WIDE>::SMEM;
  static size_t attr[64] = {};
  {
    cudaError_t e = ensure_smem((const void*)gemm2_bf16_tn_kernel<BN, EPI, WIDE>, smem, attr);
    if (e != cudaSuccess) {
      snprintf(g_err, sizeof g_err, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
      return -4;
    }
  }
  launch_pdl(gemm2_bf16_tn_kernel<BN, EPI, WIDE>, dim3(p->grid), dim3(kThreads), smem, s, p->tmA, p->tmB,
             p->tmO, p->tmR, p->tmO2, p->M, p->N, p->K, p->ep);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof g_err, "gemm2 launch: %s", cudaGetErrorString(e));
    return -4;
  }
  return 0;
}

template <int BN, int EPI>
static int launch_t2(const GemmPlan* p, cudaStream_t s) {
  if constexpr (BN == 192 && (EPI == EPI_RESID_RED || EPI == EPI_BF16))
    if (p->wide) return launch_t2w<BN, EPI, 2>(p, s);
  return launch_t2w<BN, EPI, 1>(p, s);
}

template <int BN, int EPI>
static int launch_t(const GemmPlan* p, cudaStream_t s) {
  if (p->two_cta) return launch_t2<BN, EPI>(p, s);
  constexpr int smem = GemmCfg<BN, EPI>::SMEM;
  static size_t attr[64] = {};
  {
    cudaError_t e = ensure_smem((const void*)gemm_bf16_tn_kernel<BN, EPI>, smem, attr);
    if (e != cudaSuccess) {
      snprintf(g_err, sizeof g_err, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
      return -4;
    }
  }
  launch_pdl(gemm_bf16_tn_kernel<BN, EPI>, dim3(p->grid), dim3(kThreads), smem, s, p->tmA, p->tmB,
             p->tmO, p->tmR, p->tmO2, p->M, p->N, p->K, p->ep);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof g_err, "gemm launch: %s", cudaGetErrorString(e));
    return -4;
  }
  return 0;
}

int gemm_plan_launch(const GemmPlan* p, cudaStream_t s) {
  // a plan whose exchange was attached after it was built (ddit_request_set_peers sets ep.xch
  // on the fc2 plans) needs the load / update / store epilogue: its rows go to their owners
  const int epi = p->epi == EPI_RESID_RED && (p->ep.xch || p->ep.out2) ? EPI_RESID : p->epi;
  switch (epi) {
    case EPI_QKV: return p->bn == 240 ? launch_t<240, EPI_QKV>(p, s) : launch_t<144, EPI_QKV>(p, s);
    case EPI_BF16:
      switch (p->bn) {
        case 96: return launch_t<96, EPI_BF16>(p, s);
        case 128: return launch_t<128, EPI_BF16>(p, s);
        case 192: return launch_t<192, EPI_BF16>(p, s);
        case 256: return launch_t<256, EPI_BF16>(p, s);
      }
      break;
    case EPI_GELU_BF16:
      switch (p->bn) {
        case 96: return launch_t<96, EPI_GELU_BF16>(p, s);
        case 128: return launch_t<128, EPI_GELU_BF16>(p, s);
        case 192: return launch_t<192, EPI_GELU_BF16>(p, s);
        case 256: return launch_t<256, EPI_GELU_BF16>(p, s);
      }
      break;
    case EPI_RESID:
      switch (p->bn) {
        case 96: return launch_t<96, EPI_RESID>(p, s);
        case 128: return launch_t<128, EPI_RESID>(p, s);
        case 192: return launch_t<192, EPI_RESID>(p, s);
        case 256: return launch_t<256, EPI_RESID>(p, s);
      }
      break;
    case EPI_RESID_RED:
      switch (p->bn) {
        case 96: return launch_t<96, EPI_RESID_RED>(p, s);
        case 128: return launch_t<128, EPI_RESID_RED>(p, s);
        case 192: return launch_t<192, EPI_RESID_RED>(p, s);
        case 256: return launch_t<256, EPI_RESID_RED>(p, s);
      }
      break;
    case EPI_RESID_COPY:
      switch (p->bn) {
        case 128: return launch_t<128, EPI_RESID_COPY>(p, s);
        case 192: return launch_t<192, EPI_RESID_COPY>(p, s);
        case 256: return launch_t<256, EPI_RESID_COPY>(p, s);
      }
      break;
    case EPI_F32:
      switch (p->bn) {
        case 96: return launch_t<96, EPI_F32>(p, s);
        case 128: return launch_t<128, EPI_F32>(p, s);
        case 192: return launch_t<192, EPI_F32>(p, s);
        case 256: return launch_t<256, EPI_F32>(p, s);
      }
      break;
  }
  snprintf(g_err, sizeof g_err, "epilogue %d not instantiated for BN %d", p->epi, p->bn);
  return -2;
}

}  // namespace ddit
#ifdef DDIT_EPI_TRACE
extern "C" __attribute__((visibility("default"))) int ddit_debug_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, ddit::g_epi_trace, sizeof(unsigned long long) * (n < 1024 ? n : 1024));
}
#endif
