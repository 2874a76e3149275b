// Temporal self-attention (T <= 64 frames) on tcgen05 /
// TMEM, fed by cp.async.
//
// The temporal sequences of the DDiT step are the T frames of one token position: rows
// base + t*tok of the token-major QKV matrix, i.e. one (batch, position, head) is a tiny T x T
// problem. A work unit packs HG heads of ONE position into a 128-row MMA tile, rows
// r = i * R + t for head hg * HG + i (R = 16 for T <= 16, 32 for T <= 32, 64 for T <= 64; HG = 128 / R).
//
//   loads     : four loader warps copy the unit's q / k / v slices with 16 B cp.async straight
//               into the 128B-swizzled (columns 0..63) and 32B-swizzled (64..79) K-major operand
//               layouts. A (frame, operand) row slice of a unit is HG adjacent 144 B head slices
//               = one contiguous 1152 B (T <= 16) / 576 B run, and the CTAs holding the other head
//               groups of the position read the rest of the same 6912 B QKV rows at the same
//               time. (A TMA version -- one 5-D box per head -- moved the same bytes at only
//               2.7 TB/s: a box of 30 rows x 128 B scattered 11-25 MB apart keeps too few bytes in
//               flight.) Rows t >= T and columns 72..79 are zeroed once and never written.
//   S = Q K^T : one M128 N128 tile (5 k16 MMAs). Only its R x R diagonal blocks are meaningful
//               (block-diagonal mask); the tensor core does HG x the useful work, which costs
//               nothing here: the kernel is HBM-bound (q, k, v read once, o written once).
//   softmax   : one row per thread, its R scores from one tcgen05.ld; max, exp2, row sum in fp32.
//   P         : bf16 into TMEM (tcgen05.st, 16 columns per warp); the off-diagonal blocks are
//               zeroed once at kernel start and never written again.
//   O = P V   : tcgen05.mma with A (= P) from TMEM, V an MN-major B operand from shared memory.
//   epilogue  : O / l -> bf16 -> shared staging -> one 5-D TMA store per head {72, R frames}
//               (asynchronous: the softmax warps do not wait for the LSU behind the loaders).
//
// Persistent CTAs (grid = #SMs) take contiguous ranges of units (head group fastest). Warp roles (384 threads): 0-3
// loaders (3-stage ring, two units in flight), 4 QK issuer, 6 PV issuer, 5 TMEM allocator,
// 8-11 softmax + epilogue (the epilogue of unit n-1 runs after P of
// unit n is handed to the tensor core). TMEM: S double-buffered [0, 256), O double-buffered at
// 256 / 352, P at [448, 512).
#include "common.cuh"
#include "ddit.h"
#include "capi_internal.h"
#include "temporal_plan.cuh"

#include <cstring>

namespace ddit {
// DDIT_TA_TRACE (experiment builds only): SM-clock timeline of CTA 0, 8 slots per unit --
// 0 loads issued, 1 loads landed, 2 QK issued, 3 S read, 4 P stored, 5 PV issued, 6 epilogue done.
#ifdef DDIT_TA_TRACE
__device__ unsigned long long g_ta_trace[1024];
#define TA_TRACE(idx) \
  do {                \
    if (blockIdx.x == 0) g_ta_trace[(idx) & 1023] = clock64(); \
  } while (0)
#else
#define TA_TRACE(idx) \
  do {                \
  } while (0)
#endif
namespace ta {
constexpr int THREADS = 384;
constexpr int STAGES = 3;
constexpr int BOXA = 16384, BOXB = 4096, OPND = BOXA + BOXB;  // one 128-row operand (64 + 16 cols)
constexpr int STAGE = 3 * OPND;                                // Q, K, V
constexpr int OST = 128 * 144;                                 // O staging (72 bf16 per row)
constexpr int OFF_O = STAGES * STAGE;
constexpr int OFF_BAR = OFF_O + 2 * OST;
constexpr int SMEM = 1024 + OFF_BAR + 32 * 8;
constexpr uint32_t TM_S = 0, TM_O0 = 256, TM_O1 = 352, TM_P = 448;
static_assert(SMEM <= 232448, "temporal attention smem");

DDIT_DEV void tma_store_5d(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3,
                           int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(m)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
DDIT_DEV void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// smem matrix descriptor: start, LBO (bytes), SBO (bytes), layout (2 = SW128, 6 = SW32)
DDIT_DEV uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn_major ? (1u << 16) : 0u) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// D[tmem] (+)= A[tmem] * B[smem]: A (M x 16, bf16 packed two per 32-bit column) from TMEM.
DDIT_DEV void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t id,
                      uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(id), "r"(accumulate));
}
DDIT_DEV void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
DDIT_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
DDIT_DEV void st_shared_u4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
}  // namespace ta

// unit -> (head group, position in the batch, batch), head group fastest
struct TaUnit {
  int hg, pos, b;
};
DDIT_DEV TaUnit ta_unit(int u, const TemporalParams& p) {
  TaUnit x;
  x.hg = u % p.groups;
  const int r = u / p.groups;
  x.pos = r % p.inner;
  x.b = r / p.inner;
  return x;
}

template <int R>
__global__ void __launch_bounds__(ta::THREADS, 1)
    temporal_tc_kernel(const __grid_constant__ TemporalParams p) {
  if (threadIdx.x == 0) tma_prefetch_desc(&p.tmO);
  using namespace ta;
  constexpr int HG = 128 / R;  // heads per unit
  extern __shared__ uint8_t ta_smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ta_smem_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint64_t* st_full = bars + 0;   // [STAGES]
  uint64_t* st_empty = bars + 3;  // [STAGES]
  uint64_t* s_full = bars + 6;    // [2]
  uint64_t* s_free = bars + 8;    // [2]
  uint64_t* pv_done = bars + 10;  // [2]
  uint64_t* o_free = bars + 12;   // [2]
  uint64_t* p_full = bars + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = warp_id(), lane = lane_id();
  const int n_units = p.groups * p.inner * p.batches;
  // each CTA takes a contiguous range of units: the head groups of a position (the rest of its
  // QKV rows) run back to back on the same SM
  const int u_lo = (int)((long long)n_units * blockIdx.x / gridDim.x);
  const int u_hi = (int)((long long)n_units * (blockIdx.x + 1) / gridDim.x);
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&st_full[i], 4);
      mbar_init(&st_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
      mbar_init(&pv_done[i], 1);
      mbar_init(&o_free[i], 4);
    }
    mbar_init(p_full, 4);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  if (threadIdx.x == 0) TA_TRACE(1023);

  if (warp < 4) {  // ------------------------------------------------------------- loaders
    const int tid = threadIdx.x;  // 0..127
    // zero what the copies never write, once: the 32B-swizzled columns 72..79 of every row and
    // the rows t >= T of every head block -- or everything when the last head group is partial
    // (its missing heads' V rows must be finite: P = 0 times V in the PV MMA)
    if (p.heads % HG)
      for (int k = tid; k < STAGES * STAGE / 16; k += 128) ta::st_shared_u4(smem_u32(sm) + k * 16, 0u, 0u, 0u, 0u);
    for (int k = tid; k < STAGES * 3 * 128; k += 128) {
      const int r = k & 127;
      ta::st_shared_u4(smem_u32(sm) + (k >> 7) * OPND + BOXA + r * 32 + ((((r >> 2) & 1) ^ 1) << 4),
                       0u, 0u, 0u, 0u);
    }
    const int pad = R - p.T;
    for (int k = tid; k < STAGES * 3 * HG * pad * 9; k += 128) {
      const int c = k % 9, q2 = k / 9;
      const int r = (q2 % (HG * pad)) / pad * R + p.T + q2 % pad, op = q2 / (HG * pad);
      ta::st_shared_u4(smem_u32(sm) + op * OPND + (c < 8 ? r * 128 + c * 16 : BOXA + r * 32 + (((r >> 2) & 1) << 4)),
                       0u, 0u, 0u, 0u);
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");  // zeros in place before any copy lands
    // a (operand, frame) run of a unit is HG head slices of 144 B = CH 16 B chunks, contiguous in
    // the QKV row; lane chunk j of a run is chunk lane + 32 j (head i_j, column chunk c_j)
    constexpr int CH = 9 * HG, NJ = (CH + 31) / 32;
    int lsrc[NJ], ldst[NJ], lc[NJ], li[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int ch = lane + 32 * j;
      li[j] = ch < CH ? ch / 9 : HG;  // HG: no chunk
      lc[j] = ch % 9;
      lsrc[j] = li[j] * 72 + lc[j] * 8;
      ldst[j] = lc[j] < 8 ? li[j] * R * 128 : BOXA + li[j] * R * 32;
    }
    const int nrun = 3 * p.T;
    int n = 0;
    for (int u = u_lo; u < u_hi; ++u, ++n) {
      const TaUnit x = ta_unit(u, p);
      const int st = n % STAGES;
      if (n >= STAGES) mbar_wait(&st_empty[st], ((n / STAGES) - 1) & 1);
      const uint32_t buf = smem_u32(sm + st * STAGE);
      const __nv_bfloat16* base =
          p.qkv + ((size_t)x.b * p.outer + x.pos) * p.ld + x.hg * HG * 72;
      const int nh = min(HG, p.heads - x.hg * HG);
      for (int run = warp; run < nrun; run += 4) {  // warp w: runs w, w + 4, ...
        const int op = (run >= p.T) + (run >= 2 * p.T), t = run - op * p.T;
        const __nv_bfloat16* rs = base + (size_t)t * p.tok_ld + op * p.heads * 72;
        const uint32_t rd = buf + op * OPND;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          if (li[j] >= nh) continue;
          const uint32_t off = lc[j] < 8 ? t * 128 + ((lc[j] ^ (t & 7)) << 4) : t * 32 + (((t >> 2) & 1) << 4);
          ta::cp_async16(rd + ldst[j] + off, rs + lsrc[j]);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (tid == 0) TA_TRACE(8 * n + 0);
      if (n >= 1) {  // the previous unit's copies landed: hand its stage to the tensor core
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (tid == 0) TA_TRACE(8 * (n - 1) + 1);
        if (lane == 0) mbar_arrive(&st_full[(n - 1) % STAGES]);
      }
    }
    if (n >= 1) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&st_full[(n - 1) % STAGES]);
    }
    if (warp == 0 && lane == 0) pdl_trigger();
  } else if (warp == 4) {  // -------------------------------------------------- QK issuer
    // QK and PV are issued by different warps: PV of unit n goes out as soon as its P is in
    // TMEM, never behind the loads of unit n + 1 (which QK of n + 1 waits for)
    constexpr uint32_t id_qk = ta::idesc(128, 128, false);
    int n = 0;
    for (int u = u_lo; u < u_hi; ++u, ++n) {
      const int st = n % STAGES, b = n & 1;
      mbar_wait(&st_full[st], (n / STAGES) & 1);
      if (n >= 2) mbar_wait(&s_free[b], ((n - 2) >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t qa = smem_u32(sm + st * STAGE), ka = qa + OPND;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16_ss(tmem + TM_S + 128 * b, ta::sdesc(qa + 32 * k, 16, 1024, 2),
                       ta::sdesc(ka + 32 * k, 16, 1024, 2), id_qk, k > 0);
        umma_bf16_ss(tmem + TM_S + 128 * b, ta::sdesc(qa + BOXA, 16, 256, 6),
                     ta::sdesc(ka + BOXA, 16, 256, 6), id_qk, 1);
        umma_commit(&s_full[b]);
        TA_TRACE(8 * n + 2);
      }
      __syncwarp();
    }
  } else if (warp == 6) {  // -------------------------------------------------- PV issuer
    constexpr uint32_t id_pv64 = ta::idesc(128, 64, true);
    constexpr uint32_t id_pv16 = ta::idesc(128, 16, true);
    int n = 0;
    for (int u = u_lo; u < u_hi; ++u, ++n) {
      const int st = n % STAGES, b = n & 1;
      mbar_wait(p_full, n & 1);  // P of unit n in TMEM (its softmax read S: QK of n is complete)
      if (n >= 2) mbar_wait(&o_free[b], ((n - 2) >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t va = smem_u32(sm + st * STAGE + 2 * OPND), vb = va + BOXA;
        const uint32_t o_tm = tmem + (b ? TM_O1 : TM_O0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // 16 keys per step: P columns 8 kk .. 8 kk + 7
          ta::umma_ts(o_tm, tmem + TM_P + 8 * kk, ta::sdesc(va + kk * 2048, 8192, 1024, 2), id_pv64,
                      kk > 0);
          ta::umma_ts(o_tm + 64, tmem + TM_P + 8 * kk, ta::sdesc(vb + kk * 512, 8192, 256, 6), id_pv16,
                      kk > 0);
        }
        umma_commit(&pv_done[b]);
        umma_commit(&st_empty[st]);  // Q, K (QK done before the softmax) and V of unit n consumed
        TA_TRACE(8 * n + 5);
      }
      __syncwarp();
    }
  } else if (warp >= 8) {  // ---------------------------------------- softmax + epilogue
    const int q = warp & 3;  // TMEM lane quarter
    const int row = q * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
    {  // P: zero this warp's 64 columns once (only the diagonal blocks are rewritten)
      uint32_t z[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll
      for (int c = 0; c < 64; c += 16) ta::tmem_st16(lane_base + TM_P + c, z);
      ta::tmem_st_wait();
    }
    // row r = head * R + t; its keys are S columns [R * (r / R), + R), inside the warp's
    // 32 columns [32 q, 32 q + 32)
    auto epilogue = [&](int m, float l, const TaUnit& x) {
      const int b = m & 1;
      tc_fence_after();
      uint32_t o[80];
      const uint32_t o_tm = lane_base + (b ? TM_O1 : TM_O0);
      tmem_ld_32x32b_x32(o_tm, *reinterpret_cast<uint32_t(*)[32]>(o));
      tmem_ld_32x32b_x32(o_tm + 32, *reinterpret_cast<uint32_t(*)[32]>(o + 32));
      tmem_ld_32x32b_x16(o_tm + 64, o + 64);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 31) mbar_arrive_relaxed(&o_free[b]);
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const int sb = m & 1;
      uint8_t* stg = sm + OFF_O + sb * OST;
      if (row == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");  // this staging buffer's last stores read it
      const uint32_t ob = smem_u32(stg) + row * 144;
#pragma unroll
      for (int c = 0; c < 9; ++c)
        ta::st_shared_u4(ob + c * 16, pack_bf16(__uint_as_float(o[8 * c + 0]) * inv, __uint_as_float(o[8 * c + 1]) * inv),
                         pack_bf16(__uint_as_float(o[8 * c + 2]) * inv, __uint_as_float(o[8 * c + 3]) * inv),
                         pack_bf16(__uint_as_float(o[8 * c + 4]) * inv, __uint_as_float(o[8 * c + 5]) * inv),
                         pack_bf16(__uint_as_float(o[8 * c + 6]) * inv, __uint_as_float(o[8 * c + 7]) * inv));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (row == 0) {  // one TMA store per head: its R x 72 block (frames >= T clip)
        const int nh = min(HG, p.heads - x.hg * HG);
        for (int i = 0; i < nh; ++i) ta::tma_store_5d(&p.tmO, stg + i * R * 144, 0, x.hg * HG + i, 0, x.pos, x.b);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      if (row == 0) TA_TRACE(8 * m + 6);
    };
    int n = 0;
    float l_prev = 0.f;
    TaUnit x_prev{0, 0, 0};
    for (int u = u_lo; u < u_hi; ++u, ++n) {
      const int b = n & 1;
      mbar_wait(&s_full[b], (n >> 1) & 1);
      tc_fence_after();
      // the row's R keys: S columns [R (row / R), + R) -- inside the warp's 32 columns for R <= 32,
      // the 64 columns of its head block for R = 64
      constexpr int NL = R == 64 ? 64 : 32;
      uint32_t s[NL];
      const uint32_t scol = R == 64 ? 64u * (q >> 1) : 32u * q;
      tmem_ld_32x32b_x32(lane_base + TM_S + 128 * b + scol, *reinterpret_cast<uint32_t(*)[32]>(s));
      if constexpr (R == 64)
        tmem_ld_32x32b_x32(lane_base + TM_S + 128 * b + scol + 32, *reinterpret_cast<uint32_t(*)[32]>(s + 32));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 31) mbar_arrive_relaxed(&s_free[b]);
      if (row == 0) TA_TRACE(8 * n + 3);
      float v[R];
      if constexpr (R == 16) {
        const bool hi = lane >= 16;
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(hi ? s[16 + j] : s[j]);
      } else {
#pragma unroll
        for (int j = 0; j < R; ++j) v[j] = __uint_as_float(s[j]);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (j < p.T) mx = fmaxf(mx, v[j]);
      const float ms = mx * p.scale_log2;
      float l = 0.f;
      uint32_t pk[R / 2];
#pragma unroll
      for (int j = 0; j < R; j += 2) {
        const float e0 = j < p.T ? exp2f(fmaf(v[j], p.scale_log2, -ms)) : 0.f;
        const float e1 = j + 1 < p.T ? exp2f(fmaf(v[j + 1], p.scale_log2, -ms)) : 0.f;
        l += e0 + e1;
        pk[j / 2] = pack_bf16(e0, e1);
      }
      constexpr int NW = R == 64 ? 32 : 16;  // packed P columns this warp writes
      uint32_t w[NW];
      if constexpr (R == 16) {
        const bool hi = lane >= 16;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          w[i] = hi ? 0u : pk[i];
          w[8 + i] = hi ? pk[i] : 0u;
        }
      } else {
#pragma unroll
        for (int i = 0; i < NW; ++i) w[i] = pk[i];
      }
      // the previous unit's PV has read P (and produced its O)
      if (n >= 1) mbar_wait(&pv_done[(n - 1) & 1], ((n - 1) >> 1) & 1);
      tc_fence_after();
      if constexpr (R == 64) {
        ta::tmem_st16(lane_base + TM_P + 32 * (q >> 1), w);
        ta::tmem_st16(lane_base + TM_P + 32 * (q >> 1) + 16, w + 16);
      } else {
        ta::tmem_st16(lane_base + TM_P + 16 * q, w);
      }
      ta::tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 31) mbar_arrive(p_full);
      if (row == 0) TA_TRACE(8 * n + 4);
      const TaUnit x = ta_unit(u, p);
      if (n >= 1) epilogue(n - 1, l_prev, x_prev);
      l_prev = l;
      x_prev = x;
    }
    if (n >= 1) {
      mbar_wait(&pv_done[(n - 1) & 1], ((n - 1) >> 1) & 1);
      epilogue(n - 1, l_prev, x_prev);
    }
    if (row == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ------------------------------------------------------------------ host
typedef CUresult (*PFN_encode_ta)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encode_ta ta_encoder() {
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    return reinterpret_cast<PFN_encode_ta>(ptr);
  return nullptr;
}
int temporal_plan_init(TemporalPlan* tp, const ddit_attn* a) {
  const int C = a->heads * a->head_dim;
  const auto* q = static_cast<const __nv_bfloat16*>(a->q);
  const int inner = a->q_inner > 1 ? a->q_inner : 1;
  if (a->head_dim != 72 || a->Lq != a->Lk || a->Lq < 1 || a->Lq > 64 || a->ldq != 3 * C ||
      static_cast<const __nv_bfloat16*>(a->k) != q + C ||
      static_cast<const __nv_bfloat16*>(a->v) != q + 2 * C || a->ldk != a->ldq ||
      a->ldv != a->ldq || (a->q_inner > 1 && a->q_inner_stride != 1) || a->kv_tok != a->q_tok ||
      a->kv_outer != a->q_outer || a->kv_inner != a->q_inner || a->num_seqs % inner ||
      a->ldo % 8 || (reinterpret_cast<uintptr_t>(a->q) & 15) ||
      (reinterpret_cast<uintptr_t>(a->o) & 15)) {
    set_error("temporal attention: needs one QKV matrix, T <= 64, shared q/kv index map");
    return DDIT_E_INVALID;
  }
  memset(tp, 0, sizeof *tp);
  const int T = a->Lq;
  const int R = T <= 16 ? 16 : T <= 32 ? 32 : 64, HG = 128 / R;
  const int batches = a->num_seqs / inner;
  {
    static PFN_encode_ta enc = ta_encoder();
    cuuint64_t dims[5] = {72, (cuuint64_t)a->heads, (cuuint64_t)T, (cuuint64_t)inner, (cuuint64_t)batches};
    cuuint64_t strides[4] = {144, (cuuint64_t)a->q_tok * a->ldo * 2, (cuuint64_t)a->ldo * 2,
                             (cuuint64_t)a->q_outer * a->ldo * 2};
    cuuint32_t box[5] = {72, 1, (cuuint32_t)R, 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    if (!enc || enc(&tp->p.tmO, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, a->o, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("temporal attention: cuTensorMapEncodeTiled failed");
      return DDIT_E_TMA;
    }
  }
  tp->p.qkv = q;
  tp->p.ld = a->ldq;
  tp->p.tok_ld = (long long)a->q_tok * a->ldq;
  tp->p.outer = a->q_outer;
  tp->p.T = T;
  tp->p.heads = a->heads;
  tp->p.groups = (a->heads + HG - 1) / HG;
  tp->p.inner = inner;
  tp->p.batches = batches;
  tp->p.scale_log2 = a->scale * 1.4426950408889634f;
  tp->R = R;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int units = tp->p.groups * tp->p.inner * tp->p.batches;
  tp->grid = dim3(units < sms ? units : sms, 1, 1);
  return DDIT_OK;
}

int temporal_plan_launch(const TemporalPlan* tp, cudaStream_t s) {
  static size_t attr[3][64] = {};
  auto kern = tp->R == 16 ? temporal_tc_kernel<16> : tp->R == 32 ? temporal_tc_kernel<32> : temporal_tc_kernel<64>;
  ensure_smem((const void*)kern, ta::SMEM, attr[tp->R == 16 ? 0 : tp->R == 32 ? 1 : 2]);
  launch_pdl(kern, tp->grid, dim3(ta::THREADS), ta::SMEM, s, tp->p);
  return check_cuda("temporal_tc_kernel");
}

int temporal_attention_launch(const ddit_attn* a, cudaStream_t s) {
  TemporalPlan tp;
  int rc = temporal_plan_init(&tp, a);
  if (rc) return rc;
  return temporal_plan_launch(&tp, s);
}

}  // namespace ddit

extern "C" DDIT_API int ddit_attention_temporal(const ddit_attn* a, void* stream) {
  return ddit::temporal_attention_launch(a, static_cast<cudaStream_t>(stream));
}

#ifdef DDIT_TA_TRACE
extern "C" __attribute__((visibility("default"))) int ddit_ta_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, ddit::g_ta_trace, sizeof(unsigned long long) * (n < 1024 ? n : 1024));
}
#endif
