// tcgen05 / TMEM flash attention (forward, non-causal, head_dim 72) for the STDiT3 spatial
// and cross attention.
//
// One CTA = one work unit (sequence, head, PAIR of 128-query tiles); the two Q tiles ping-pong
// on the tensor core so that one tile's softmax always overlaps the other tile's MMAs.
// Warp roles (384 threads):
//   warp 0      : TMA producer. Q/K/V come straight out of the token-major QKV (or q / kv)
//                 matrices through 4-D tensor maps {72, head slot, token, sequence}: the token
//                 dimension is clipped at the sequence length, so ragged tiles zero-fill on load
//                 and clip on store. head_dim 72 is split into a 64-column 128B-swizzled box and
//                 a 16-column 32B-swizzled box whose columns 72..79 fall outside the map (zeros).
//   warps 1, 3  : MMA issuers (one thread each; warp 1 for Q tile 0, warp 3 for Q tile 1). Per
//                 K/V tile j: S_g = Q_g K_j^T (M128 N128, K = 4 x16 SW128 + 1 x16 SW32) as soon
//                 as group g holds S_{j-1} in registers, then O_g += P_g V_{j-1} (V as an MN-major
//                 B operand, N64 SW128 + N16 SW32, 8 k-steps of 16 keys): the scores of tile j
//                 are computed while the softmax of tile j-1 runs; the groups never wait on
//                 each other.
//   warp 2      : TMEM allocator.
//   warps 4-7   : softmax of Q tile 0 of the unit, warps 8-11: of Q tile 1. One query row per
//                 thread (= TMEM lane), all 128 keys of a tile in registers (setmaxnreg 200), so
//                 no cross-warp exchange: online softmax in fp32 with exp2, lazy O rescaling
//                 (only when the running max grows by > 2^8), P written as bf16 into
//                 128B-swizzled smem (the A operand of PV); final O / l -> bf16 -> smem (the
//                 tile's P buffer) -> TMA store.
// Persistent: grid = #SMs, each CTA walks units (q-tile pair fastest, so concurrent CTAs share
// K/V in L2); Q is double-buffered per softmax group, K and V stream through their own rings
// across units. TMEM: S0 [0,128), S1 [128,256), O0 [256,336), O1 [336,416), P0 [416,464), P1 [464,512).
#include "common.cuh"
#include "ddit.h"
#include "capi_internal.h"
#include "fmha_plan.cuh"

#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>

namespace ddit {

// DDIT_FMHA_TRACE (experiment builds only): SM-clock timeline of CTA 0 -- per softmax group and
// tile: S ready, MUFU token taken, exps done, P buffer free, P stored; per unit: O ready, O
// stored; per MMA warp and tile: QK issued, PV issued. Read back with ddit_fmha_trace().
#ifdef DDIT_FMHA_TRACE
__device__ unsigned long long g_fm_trace[2048];
#define FM_TRACE(idx) \
  do {                \
    if (blockIdx.x == 0) g_fm_trace[(idx) & 2047] = clock64(); \
  } while (0)
#else
#define FM_TRACE(idx) \
  do {                \
  } while (0)
#endif

namespace fm {
constexpr int BQ = 128, BKV = 128, THREADS = 384, KST = 2, VST = 2;
constexpr int QA = 16384, QB = 4096, QT = QA + QB;  // one Q tile: 64-col SW128 + 16-col SW32 boxes
constexpr int KA = 16384, KB = 4096, VA = 16384, VB = 4096;
constexpr int PBUF = 2 * 16384;                    // P of one Q tile: two 64-key SW128 regions
constexpr int OFF_Q = 0;                           // [2 groups][2 buffers] Q tiles
constexpr int OFF_K = OFF_Q + 4 * QT;              // KST K stages
constexpr int OFF_V = OFF_K + KST * (KA + KB);     // VST V stages
constexpr int OFF_P = OFF_V + VST * (VA + VB);     // P per group (also its O store staging)
constexpr int OFF_BAR = OFF_P + 2 * PBUF;
constexpr int NBAR = 32;
constexpr int SMEM = 1024 + OFF_BAR + NBAR * 8 + 16;
#ifndef DDIT_FMHA_PTMEM
#define DDIT_FMHA_PTMEM 1
#endif
#if DDIT_FMHA_PTMEM
// group g: S at TM_S0 + 128 g, O at TM_O0 + 80 g, keys 0..95 of P (bf16, two per column) at
// TM_P0 + 48 g; keys 96..127 of P stay in shared memory
constexpr uint32_t TM_S0 = 0, TM_O0 = 256, TM_OSTEP = 80, TM_P0 = 416, TM_PSTEP = 48;
constexpr int P_TM_CHUNKS = 12;  // 8-key chunks of P held in TMEM
#else
constexpr uint32_t TM_S0 = 0, TM_O0 = 256, TM_OSTEP = 128;  // group g: S at TM_S0 + 128 g, O at TM_O0 + 128 g
constexpr int P_TM_CHUNKS = 0;
#endif
constexpr float RESCALE_LOG2 = 8.0f;
static_assert(SMEM <= 232448, "fmha smem");
}  // namespace fm


DDIT_DEV void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                          int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
DDIT_DEV void tma_store_4d(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
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
// D[tmem] (+)= A[tmem] * B[smem] (A: M x 16 bf16, two per 32-bit TMEM column)
DDIT_DEV void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                      uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn_major ? (1u << 16) : 0u) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

DDIT_DEV void tmem_ld32(uint32_t taddr, uint32_t* r) {
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
DDIT_DEV void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
DDIT_DEV void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
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
DDIT_DEV void tmem_ld_32x32b_x8_fm(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
// 2^x on the FMA pipe (x <= 0 here): 2^floor(x) * p(frac), p a degree-4 least-squares polynomial of
// 2^f on [0, 1) (rel. err 5e-6 << bf16), exponent inserted with an integer add.
DDIT_DEV float poly_exp2(float x) {
  x = fmaxf(x, -127.f);
  const float fl = floorf(x);
  const float f = x - fl;
  float p = 1.351155e-2f;
  p = fmaf(p, f, 5.198954e-2f);
  p = fmaf(p, f, 2.4150888e-1f);
  p = fmaf(p, f, 6.9297426e-1f);
  p = fmaf(p, f, 1.00000526f);
  return __int_as_float(__float_as_int(p) + (static_cast<int>(fl) << 23));
}
// Blackwell packed fp32: two FMAs / adds per instruction, and a 3-input max.
DDIT_DEV void ffma2(float& d0, float& d1, float a0, float a1, float b, float c) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\tmov.b64 rc, {%5, %5};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b), "f"(c));
}
DDIT_DEV void fadd2(float& a0, float& a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb;\n\tmov.b64 ra, {%0, %1};\n\tmov.b64 rb, {%2, %3};\n\t"
      "add.rn.f32x2 ra, ra, rb;\n\tmov.b64 {%0, %1}, ra;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(b0), "f"(b1));
}
DDIT_DEV float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
DDIT_DEV void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// Two 2^x on the FMA pipe (x <= ~8; clamped at -127): round-to-nearest split x = j + f through the
// 1.5 * 2^23 magic add, f in [-0.5, 0.5], cubic minimax p(f) (rel. err 1.4e-4 << bf16 ulp), then j
// added into the exponent field with one integer op -- offloads part of the exps from MUFU.
DDIT_DEV float2 exp2_poly_x2(float x0, float x1) {
  const float2 x = make_float2(fmaxf(x0, -127.f), fmaxf(x1, -127.f));
  const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 q = __ffma2_rn(make_float2(0.05502926645f, 0.05502926645f), f,
                        make_float2(0.24225698193f, 0.24225698193f));
  q = __ffma2_rn(q, f, make_float2(0.69325305500f, 0.69325305500f));
  q = __ffma2_rn(q, f, make_float2(0.99995133866f, 0.99995133866f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}
// chunks (8 keys each) of a full tile whose exps run on the FMA pipe instead of MUFU: every
// POLY-th chunk (POLY = 0: none)
template <int POLY>
__host__ __device__ constexpr bool poly_chunk(int c) { return POLY > 0 && c % POLY == POLY - 1; }
// 1 / x for x > 0 on the FMA pipe (bit-trick seed + 3 Newton steps, rel. err ~1e-7): MUFU.RCP
// would queue behind the other softmax group's exps
DDIT_DEV float rcp_fma(float x) {
  float r = __int_as_float(0x7EF311C7 - __float_as_int(x));
  r = r * fmaf(-x, r, 2.f);
  r = r * fmaf(-x, r, 2.f);
  r = r * fmaf(-x, r, 2.f);
  return r;
}
DDIT_DEV float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Work-unit walk of a persistent CTA: unit u = blockIdx.x, +gridDim.x, ... decomposed as
// (q-tile pair fastest, head, sequence) -- pair fastest so concurrent CTAs share K/V in L2. The
// coordinates advance by a mixed-radix add: no integer division inside the loops (it would go
// through MUFU.RCP, queued behind the other softmax group's exps).
struct UnitWalk {
  int u, pr, head, seq;
  int G, pairs, heads, d_pr, d_head, d_seq;
  DDIT_DEV UnitWalk(int pairs_, int heads_) : pairs(pairs_), heads(heads_) {
    G = gridDim.x;
    u = blockIdx.x;
    pr = u % pairs;
    head = (u / pairs) % heads;
    seq = u / (pairs * heads);
    d_pr = G % pairs;
    d_head = (G / pairs) % heads;
    d_seq = G / (pairs * heads);
  }
  DDIT_DEV void next() {
    u += G;
    pr += d_pr;
    int c = pr >= pairs;
    pr -= c ? pairs : 0;
    head += d_head + c;
    c = head >= heads;
    head -= c ? heads : 0;
    seq += d_seq + c;
  }
};

template <int POLY>
__global__ void __launch_bounds__(fm::THREADS, 1)
    fmha_sm100_kernel(const __grid_constant__ CUtensorMap tmQa,
                      const __grid_constant__ CUtensorMap tmQb,
                      const __grid_constant__ CUtensorMap tmKVa,
                      const __grid_constant__ CUtensorMap tmKVb,
                      const __grid_constant__ CUtensorMap tmO,
                      const __grid_constant__ FmhaParams p) {
  using namespace fm;
  extern __shared__ uint8_t fm_smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(fm_smem_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint64_t* q_full = bars + 0;    // [group * 2 + buffer]
  uint64_t* q_empty = bars + 4;   // [group * 2 + buffer]
  uint64_t* k_full = bars + 8;    // [KST]
  uint64_t* k_empty = bars + 10;  // [KST]
  uint64_t* v_full = bars + 12;   // [VST]
  uint64_t* v_empty = bars + 14;  // [VST]
  uint64_t* s_full = bars + 16;   // [group]
  uint64_t* s_free = bars + 18;   // [group]
  uint64_t* p_full = bars + 20;   // [group]
  uint64_t* pv_done = bars + 22;  // [group]
  uint64_t* o_free = bars + 24;   // [group]
  uint64_t* exp_tok = bars + 26;  // [group]: the group may run its exps phase (MUFU turn)
  uint64_t* v_ready = bars + 28;  // [VST]: V stage landed and carries the ones column
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 30);

  const int warp = warp_id(), lane = lane_id();
  const int nk = (p.Lk + BKV - 1) / BKV;
  const int pairs = (p.q_tiles + 1) >> 1;
  const int n_units = pairs * p.heads * p.seqs;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQa);
    tma_prefetch_desc(&tmQb);
    tma_prefetch_desc(&tmKVa);
    tma_prefetch_desc(&tmKVb);
    tma_prefetch_desc(&tmO);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 2);  // released by both groups' MMA warps
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 2);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[i], 1);
      mbar_init(&o_free[i], 4);
      mbar_init(&exp_tok[i], 4);
      mbar_init(&v_ready[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  // unit -> (q-tile pair, head, sequence): see UnitWalk; each role builds its own walker after
  // its setmaxnreg, so the walk state is not live across the role split
  auto first = [&]() { return UnitWalk(pairs, p.heads); };
  auto advance = [](UnitWalk& w) { w.next(); };
  using Walk = UnitWalk;
  auto has_second = [&](const Walk& w) { return 2 * w.pr + 1 < p.q_tiles; };

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;" ::: "memory");
    if (warp == 0 && lane == 0) {  // ------------------------------------------ TMA producer
      // Loads go out in the order the MMA warps consume them -- K_j before V_{j-1} (QK_j is issued
      // before PV_{j-1}), and the next unit's Q and K_0 before this unit's last V -- so a load
      // never queues behind a V stage that frees only after a later softmax phase: the next
      // unit's first QK can issue right after this unit's last PV.
      int kc = 0, vc = 0, qc[2] = {0, 0};
      auto load_q = [&](const Walk& w) {
        const bool has1 = has_second(w);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (g == 1 && !has1) break;
          const int qi = g * 2 + (qc[g] & 1);
          mbar_wait(&q_empty[qi], ((qc[g] >> 1) & 1) ^ 1);
          uint8_t* qbuf = sm + OFF_Q + qi * QT;
          mbar_arrive_expect_tx(&q_full[qi], QT);
          tma_load_4d(qbuf, &tmQa, &q_full[qi], 0, p.q_slot + w.head, (2 * w.pr + g) * BQ, w.seq);
          tma_load_4d(qbuf + QA, &tmQb, &q_full[qi], 64, p.q_slot + w.head, (2 * w.pr + g) * BQ, w.seq);
          ++qc[g];
        }
      };
      auto load_k = [&](const Walk& w, int j) {
        const int ks = kc % KST;
        mbar_wait(&k_empty[ks], ((kc / KST) & 1) ^ 1);
        uint8_t* kb = sm + OFF_K + ks * (KA + KB);
        mbar_arrive_expect_tx(&k_full[ks], KA + KB);
        tma_load_4d(kb, &tmKVa, &k_full[ks], 0, p.k_slot + w.head, j * BKV, w.seq);
        tma_load_4d(kb + KA, &tmKVb, &k_full[ks], 64, p.k_slot + w.head, j * BKV, w.seq);
        ++kc;
      };
      auto load_v = [&](const Walk& w, int j) {
        const int vs = vc % VST;
        mbar_wait(&v_empty[vs], ((vc / VST) & 1) ^ 1);
        uint8_t* vb = sm + OFF_V + vs * (VA + VB);
        mbar_arrive_expect_tx(&v_full[vs], VA + VB);
        tma_load_4d(vb, &tmKVa, &v_full[vs], 0, p.v_slot + w.head, j * BKV, w.seq);
        tma_load_4d(vb + VA, &tmKVb, &v_full[vs], 64, p.v_slot + w.head, j * BKV, w.seq);
        ++vc;
      };
      int ul = 0;
      Walk w = first();
      if (w.u < n_units) {
        load_q(w);
        load_k(w, 0);
      }
      for (; w.u < n_units; ++ul) {
        FM_TRACE(1792 + (ul & 63) * 4 + 0);
        for (int j = 1; j < nk; ++j) {
          load_k(w, j);
          load_v(w, j - 1);
        }
        Walk wn = w;
        advance(wn);
        if (wn.u < n_units) {
          load_q(wn);
          FM_TRACE(1792 + ((ul + 1) & 63) * 4 + 1);
          load_k(wn, 0);
          FM_TRACE(1792 + ((ul + 1) & 63) * 4 + 2);
        }
        load_v(w, nk - 1);
        FM_TRACE(1792 + (ul & 63) * 4 + 3);
        w = wn;
      }
      pdl_trigger();
    } else if (warp == 1 || warp == 3) {  // ------------------------ MMA issuers, one per group
      // Each softmax group has its own issuing warp (warp 1: group 0, warp 3: group 1), so a
      // group's QK / PV go to the tensor core as soon as ITS softmax is ready, independent of the
      // other group's progress; the shared K / V stages are released by both (count-2 barriers).
      // The group's tiles form one stream across units: QK_j is issued before PV_{j-1}, and the
      // next unit's first QK before this unit's last PV, so S of the next unit is ready when the
      // softmax finishes this unit (its O epilogue runs later, inside the next unit's first tile).
      const int g = warp == 1 ? 0 : 1;
      constexpr uint32_t id_qk = idesc_f16(128, 128, false);
      constexpr uint32_t id_pv64 = idesc_f16(128, 64, true);
      constexpr uint32_t id_pv16 = idesc_f16(128, 16, true);
      const uint32_t s_tmem = tmem + TM_S0 + 128 * g, o_tmem = tmem + TM_O0 + TM_OSTEP * g;
      const uint32_t pb = smem_u32(sm + OFF_P + g * PBUF);
      int kc = 0, vc = 0, qc = 0, sn = 0, pn = 0, un = 0, upv = 0;
      auto issue_qk = [&](uint32_t qa, int j) {
        mbar_wait(&k_full[kc % KST], (kc / KST) & 1);
        if (sn > 0) mbar_wait(&s_free[g], (sn - 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t ka = smem_u32(sm + OFF_K + (kc % KST) * (KA + KB)), kb = ka + KA;
          // ragged last tile: only round16(valid) key columns (the rest of S is never read)
          const int kv16 = (min(BKV, p.Lk - j * BKV) + 15) & ~15;
          const uint32_t idq = kv16 == BKV ? id_qk : idesc_f16(128, kv16, false);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16_ss(s_tmem, sdesc(qa + 32 * k, 16, 1024, 2), sdesc(ka + 32 * k, 16, 1024, 2),
                         idq, k > 0);
          umma_bf16_ss(s_tmem, sdesc(qa + QA, 16, 256, 6), sdesc(kb, 16, 256, 6), idq, 1);
          umma_commit(&s_full[g]);
          umma_commit(&k_empty[kc % KST]);
          FM_TRACE(1024 + g * 256 + (sn & 63) * 2);
        }
        __syncwarp();
        ++sn;
        ++kc;
      };
      // O (+)= P_j V_j once the group wrote P; a unit's first PV overwrites O, so the group's
      // epilogue must have read the previous unit's O (o_free)
      auto issue_pv = [&](int j) {
        if (j == 0) {
          if (upv > 0) mbar_wait(&o_free[g], (upv - 1) & 1);
          ++upv;
        }
        mbar_wait(&v_ready[vc % VST], (vc / VST) & 1);
        mbar_wait(&p_full[g], pn & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t va = smem_u32(sm + OFF_V + (vc % VST) * (VA + VB)), vb = va + VA;
          const int ksteps = (min(BKV, p.Lk - j * BKV) + 15) >> 4;  // 16-key steps with keys
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            if (kk >= ksteps) break;
            const uint32_t acc = (j > 0 || kk > 0) ? 1u : 0u;
#if DDIT_FMHA_PTMEM
            if (kk < P_TM_CHUNKS / 2) {  // P keys 16 kk .. 16 kk + 15 from TMEM (A operand in TMEM)
              const uint32_t pa = tmem + TM_P0 + TM_PSTEP * g + 8 * kk;
              umma_ts(o_tmem, pa, sdesc(va + kk * 2048, 8192, 1024, 2), id_pv64, acc);
              umma_ts(o_tmem + 64, pa, sdesc(vb + kk * 512, 8192, 256, 6), id_pv16, acc);
              continue;
            }
#endif
            const uint64_t a = sdesc(pb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, 2);
            umma_bf16_ss(o_tmem, a, sdesc(va + kk * 2048, 8192, 1024, 2), id_pv64, acc);
            umma_bf16_ss(o_tmem + 64, a, sdesc(vb + kk * 512, 8192, 256, 6), id_pv16, acc);
          }
          umma_commit(&pv_done[g]);
          umma_commit(&v_empty[vc % VST]);
          FM_TRACE(1024 + g * 256 + (pn & 63) * 2 + 1);
        }
        __syncwarp();
        ++pn;
        ++vc;
      };
      int pend = -1;  // tile index (in its unit) of the PV still to issue
      for (Walk w = first(); w.u < n_units; advance(w)) {
        if (g == 1 && !has_second(w)) {  // no second Q tile: keep the shared K / V ring in step
          if (pend >= 0) issue_pv(pend);  // (its V stage precedes this unit's)
          pend = -1;
          for (int j = 0; j < nk; ++j, ++kc, ++vc) {
            mbar_wait(&k_full[kc % KST], (kc / KST) & 1);
            if (lane == 0) mbar_arrive(&k_empty[kc % KST]);
            mbar_wait(&v_ready[vc % VST], (vc / VST) & 1);
            if (lane == 0) mbar_arrive(&v_empty[vc % VST]);
            __syncwarp();
          }
          continue;
        }
        const int qi = g * 2 + (qc & 1);
        const uint32_t qa = smem_u32(sm + OFF_Q + qi * QT);
        if (lane == 0) FM_TRACE(1536 + g * 128 + (un & 31) * 4 + 0);
        mbar_wait(&q_full[qi], (qc >> 1) & 1);
        if (lane == 0) FM_TRACE(1536 + g * 128 + (un & 31) * 4 + 1);
        for (int j = 0; j < nk; ++j) {
          issue_qk(qa, j);
          if (pend >= 0) issue_pv(pend);
          pend = j;
        }
        ++qc;
        ++un;
      }
      if (pend >= 0) issue_pv(pend);
    } else if (warp == 2) {  // ----------------------------------- V fixup (row sums on the TC)
      // head_dim 72 leaves V columns 72..79 of every stage zero (TMA out-of-bounds fill). Writing
      // ones into column 72 makes the PV MMA produce O[:, 72] = sum_k P[:, k]: the softmax row sum
      // comes out of the tensor core in fp32, from the same bf16 P as the numerator, and the
      // softmax warps drop their per-element sum. Column 72 = element 8 of the 16-column SW32
      // tail: 16 B chunk 1 of each 32 B row, swizzled with bit 2 of the row.
      int vc = 0;
      const uint32_t tail0 = smem_u32(sm + OFF_V + VA);
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        for (int j = 0; j < nk; ++j, ++vc) {
          const int vs = vc % VST;
          mbar_wait(&v_full[vs], (vc / VST) & 1);
          const uint32_t tail = tail0 + vs * (VA + VB);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = lane + 32 * i;
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(tail + r * 32 + (((r >> 2) & 1) ? 0 : 16)),
                         "h"((unsigned short)0x3F80)
                         : "memory");  // bf16 1.0
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&v_ready[vs]);
        }
      }
    }
  } else {  // ------------------------------------------------------------ softmax groups
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;" ::: "memory");
    const int g = (warp - 4) >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t s_tm = lane_base + TM_S0 + 128 * g, o_tm = lane_base + TM_O0 + TM_OSTEP * g;
    const int bar_id = 1 + g;
    const bool elected = quarter == 0 && lane == 0;
    uint8_t* pbuf = sm + OFF_P + g * PBUF;
    int n = 0;   // tiles processed by this group
    int tk = 0;  // exps phases run under the MUFU token (tiles of units with both groups)
    int qc = 0;  // units of this group (its Q buffer of unit i is g * 2 + (i & 1))
    // The O epilogue of a unit is deferred into the next unit's first tile (after its exps), so
    // it overlaps the other group's exps phase instead of stalling the MUFU turn order. O is
    // staged in the unit's own Q buffer (its last QK completed before its last PV): once the TMA
    // store has read it, q_empty hands the buffer back to the producer.
    int e_qt = 0, e_head = 0, e_seq = 0, e_qi = -1, q_release = -1;
    auto epilogue = [&]() {
      mbar_wait(&pv_done[g], (n - 1) & 1);  // the unit's last PV (tile n-1)
      if (quarter == 0 && lane == 0) FM_TRACE(g * 512 + ((n - 1) & 63) * 8 + 5);
      tc_fence_after();
      uint32_t o[16];  // columns 64..79: O[64..71], the row sum l (ones column of V) at 72
      tmem_ld16(o_tm + 64, o);
      tmem_ld_wait();
      const float l = __uint_as_float(o[8]);
      const float inv = l > 0.f ? rcp_fma(l) : 0.f;
      uint8_t* stage = sm + OFF_Q + e_qi * QT;
      const uint32_t obase = smem_u32(stage) + row * 144;
      st_shared_u4(obase + 128, pack_bf16(__uint_as_float(o[0]) * inv, __uint_as_float(o[1]) * inv),
                   pack_bf16(__uint_as_float(o[2]) * inv, __uint_as_float(o[3]) * inv),
                   pack_bf16(__uint_as_float(o[4]) * inv, __uint_as_float(o[5]) * inv),
                   pack_bf16(__uint_as_float(o[6]) * inv, __uint_as_float(o[7]) * inv));
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        uint32_t oc[32];
        tmem_ld32(o_tm + 32 * h, oc);
        tmem_ld_wait();
        if (h == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 31) mbar_arrive_relaxed(&o_free[g]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
          st_shared_u4(obase + h * 64 + c * 16,
                       pack_bf16(__uint_as_float(oc[8 * c + 0]) * inv, __uint_as_float(oc[8 * c + 1]) * inv),
                       pack_bf16(__uint_as_float(oc[8 * c + 2]) * inv, __uint_as_float(oc[8 * c + 3]) * inv),
                       pack_bf16(__uint_as_float(oc[8 * c + 4]) * inv, __uint_as_float(oc[8 * c + 5]) * inv),
                       pack_bf16(__uint_as_float(oc[8 * c + 6]) * inv, __uint_as_float(oc[8 * c + 7]) * inv));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
      if (elected) {
        tma_store_4d(&tmO, stage, 0, p.o_slot + e_head, e_qt * BQ, e_seq);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        FM_TRACE(g * 512 + ((n - 1) & 63) * 8 + 6);
      }
      q_release = e_qi;
      e_qi = -1;
    };
    for (Walk w = first(); w.u < n_units; advance(w)) {
      const bool has1 = has_second(w);
      if (g == 1 && !has1) continue;
      const int qt = 2 * w.pr + g, head = w.head, seq = w.seq;
      float m = -INFINITY;
      for (int j = 0; j < nk; ++j, ++n) {
        const bool trc = quarter == 0 && lane == 0;
        if (trc) FM_TRACE(g * 512 + (n & 63) * 8 + 7);
        mbar_wait(&s_full[g], n & 1);
        if (trc) FM_TRACE(g * 512 + (n & 63) * 8 + 0);
        tc_fence_after();
        uint32_t s[128];
        tmem_ld32(s_tm, s);
        tmem_ld32(s_tm + 32, s + 32);
        tmem_ld32(s_tm + 64, s + 64);
        tmem_ld32(s_tm + 96, s + 96);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 31) mbar_arrive_relaxed(&s_free[g]);  // lane 0 of warp 4/8 issues the O bulk stores
        const int valid = min(BKV, p.Lk - j * BKV);
        const bool full = valid == BKV;
        float mx8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx8[e] = -INFINITY;
        if (full) {
#pragma unroll
          for (int e = 0; e < 128; e += 2)
            mx8[(e >> 1) & 7] = fmax3(mx8[(e >> 1) & 7], __uint_as_float(s[e]), __uint_as_float(s[e + 1]));
        } else {  // ragged last tile: whole 8-key chunks below `valid`, then the partial one
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            if (c * 8 >= valid) break;
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (c * 8 + e < valid) mx8[e] = fmaxf(mx8[e], __uint_as_float(s[c * 8 + e]));
          }
        }
        const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        const float m_new = fmaxf(m, mx * p.scale_log2);
        const bool resc = m_new > m + RESCALE_LOG2;
        float alpha = 1.f;
        if (resc) {
          alpha = fast_exp2(m - m_new);
          m = m_new;
        }
        // MUFU turn: the two groups' exps phases alternate (g0 tile j, g1 tile j, g0 tile j+1, ...)
        // so each runs at the full SFU rate while the other does its max / P stores / waits,
        // instead of both contending in phase
        // (the ragged last tile of a unit -- a few keys -- runs outside the turn order: both groups
        // skip it, so the alternation stays in step; cross attention 34.6 -> 34.1 us)
        if (has1 && full) mbar_wait(&exp_tok[g], (tk & 1) ^ (g == 0 ? 1 : 0));
        if (trc) FM_TRACE(g * 512 + (n & 63) * 8 + 1);
        // exps first (packed bf16 P kept in the consumed s[] registers: chunk c -> s[4c..4c+3]),
        // so the MUFU work overlaps the tensor core finishing PV_{j-1}
        const float neg_m = -m;
        if (full) {
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            float pv[8];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              float x0, x1;
              ffma2(x0, x1, __uint_as_float(s[c * 8 + e]), __uint_as_float(s[c * 8 + e + 1]),
                    p.scale_log2, neg_m);
              if (poly_chunk<POLY>(c)) {
                const float2 y = exp2_poly_x2(x0, x1);
                pv[e] = y.x;
                pv[e + 1] = y.y;
              } else {
                pv[e] = fast_exp2(x0);
                pv[e + 1] = fast_exp2(x1);
              }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) s[4 * c + e] = pack_bf16(pv[2 * e], pv[2 * e + 1]);
          }
        } else {
          // ragged last tile: PV reads only the round16(valid) keys QK wrote, so the loop leaves
          // (a real branch, not predication -- a predicated tail costs a whole tile of MUFU issue)
          // after the chunks holding them; keys in [valid, round16(valid)) get P = 0
          const int kv16 = (valid + 15) & ~15;
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            if (c * 8 >= kv16) break;
            float pv[8];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              float x0, x1;
              ffma2(x0, x1, __uint_as_float(s[c * 8 + e]), __uint_as_float(s[c * 8 + e + 1]),
                    p.scale_log2, neg_m);
              pv[e] = fast_exp2(x0);
              pv[e + 1] = fast_exp2(x1);
            }
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (c * 8 + e >= valid) pv[e] = 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) s[4 * c + e] = pack_bf16(pv[2 * e], pv[2 * e + 1]);
          }
        }
        if (trc) FM_TRACE(g * 512 + (n & 63) * 8 + 2);
        if (has1 && full) {  // hand the MUFU turn to the other group
          __syncwarp();
          if (lane == 31) mbar_arrive_relaxed(&exp_tok[g ^ 1]);
          ++tk;
        }
        if (j > 0) {
          // PV of the previous tile done: P buffer free, O complete through tile j-1
          mbar_wait(&pv_done[g], (n - 1) & 1);
          if (trc) FM_TRACE(g * 512 + (n & 63) * 8 + 3);
          if (__any_sync(0xffffffffu, resc)) {
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < 80; c += 16) {  // 16 columns at a time
              uint32_t o[16];
              tmem_ld16(o_tm + c, o);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              tmem_st16(o_tm + c, o);
            }
            tmem_st_wait();
          }
        } else if (e_qi >= 0) {
          // previous unit's O epilogue (its last PV also freed the P buffer)
          epilogue();
        }
        const uint32_t prow = smem_u32(pbuf) + (uint32_t)(row * 128);
#if DDIT_FMHA_PTMEM
        // chunks 0..11 (keys 0..95) -> TMEM columns (two bf16 per column), issued first
        tmem_st16(lane_base + TM_P0 + TM_PSTEP * g, s);
        tmem_st16(lane_base + TM_P0 + TM_PSTEP * g + 16, s + 16);
        tmem_st16(lane_base + TM_P0 + TM_PSTEP * g + 32, s + 32);
#endif
#pragma unroll
        for (int c = P_TM_CHUNKS; c < 16; ++c)  // chunk c (8 keys) -> region c / 8, 16 B swizzled
          st_shared_u4(prow + (c >> 3) * 16384 + (((c & 7) ^ (row & 7)) << 4), s[4 * c], s[4 * c + 1],
                       s[4 * c + 2], s[4 * c + 3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#if DDIT_FMHA_PTMEM
        tmem_st_wait();
#endif
        tc_fence_before();
        __syncwarp();
        if (lane == 31) mbar_arrive(&p_full[g]);  // release (P stores), from a lane without bulk copies
        if (trc) FM_TRACE(g * 512 + (n & 63) * 8 + 4);
        if (q_release >= 0) {  // the O store has read its staging: the Q buffer goes back
          if (elected) {
            bulk_wait_read0();
            mbar_arrive(&q_empty[q_release]);
          }
          q_release = -1;
        }
      }
      e_qt = qt;
      e_head = head;
      e_seq = seq;
      e_qi = g * 2 + (qc & 1);
      ++qc;
    }
    if (e_qi >= 0) epilogue();
    if (elected) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ------------------------------------------------------------------ host
typedef CUresult (*PFN_encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                               const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                               const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encode encoder() {
  static PFN_encode fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encode>(ptr);
  });
  return fn;
}

// View of a token-major bf16 matrix as {72 (d), slots, L tokens, seqs}.
static bool map4d(CUtensorMap* m, const void* base, int slots, int L, int seqs, size_t row_bytes,
                  size_t seq_bytes, int box0, CUtensorMapSwizzle sw) {
  PFN_encode enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[4] = {72, (cuuint64_t)slots, (cuuint64_t)L, (cuuint64_t)seqs};
  cuuint64_t strides[3] = {144, (cuuint64_t)row_bytes, (cuuint64_t)seq_bytes};
  cuuint32_t box[4] = {(cuuint32_t)box0, 1, 128, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Whether the tcgen05 path applies: contiguous sequences (tok == 1, inner == 1), strides and
// head offsets in whole 72-column slots, k and v in one matrix.
bool fmha_supported(const ddit_attn* a) {
  if (a->head_dim != 72) return false;
  if (a->q_tok != 1 || a->kv_tok != 1) return false;
  if ((a->q_inner > 1) || (a->kv_inner > 1)) return false;
  if (a->ldq % 72 || a->ldk % 72 || a->ldo % 72 || a->ldv != a->ldk) return false;
  const auto* k = static_cast<const __nv_bfloat16*>(a->k);
  const auto* v = static_cast<const __nv_bfloat16*>(a->v);
  if (v < k || (v - k) % 72) return false;
  auto al = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  return al(a->q) && al(a->k) && al(a->o);
}

int fmha_plan_init(FmhaPlan* fp, const ddit_attn* a) {
  if (!fmha_supported(a)) {
    set_error("fmha: layout not supported by the tcgen05 path");
    return DDIT_E_INVALID;
  }
  memset(fp, 0, sizeof *fp);
  // slot extents cover exactly the heads used (k, v share one map: v = k + v_slot slots)
  const int v_slot = (int)((static_cast<const __nv_bfloat16*>(a->v) -
                            static_cast<const __nv_bfloat16*>(a->k)) / 72);
  const int q_slots = a->heads, kv_slots = v_slot + a->heads, o_slots = a->heads;
  const size_t q_seq = (size_t)a->q_outer * a->ldq * 2, kv_seq = (size_t)a->kv_outer * a->ldk * 2;
  const size_t o_seq = (size_t)a->q_outer * a->ldo * 2;
  bool ok = map4d(&fp->tmQa, a->q, q_slots, a->Lq, a->num_seqs, (size_t)a->ldq * 2, q_seq, 64,
                  CU_TENSOR_MAP_SWIZZLE_128B) &&
            map4d(&fp->tmQb, a->q, q_slots, a->Lq, a->num_seqs, (size_t)a->ldq * 2, q_seq, 16,
                  CU_TENSOR_MAP_SWIZZLE_32B) &&
            map4d(&fp->tmKVa, a->k, kv_slots, a->Lk, a->num_seqs, (size_t)a->ldk * 2, kv_seq, 64,
                  CU_TENSOR_MAP_SWIZZLE_128B) &&
            map4d(&fp->tmKVb, a->k, kv_slots, a->Lk, a->num_seqs, (size_t)a->ldk * 2, kv_seq, 16,
                  CU_TENSOR_MAP_SWIZZLE_32B) &&
            map4d(&fp->tmO, a->o, o_slots, a->Lq, a->num_seqs, (size_t)a->ldo * 2, o_seq, 72,
                  CU_TENSOR_MAP_SWIZZLE_NONE);
  if (!ok) {
    set_error("fmha: cuTensorMapEncodeTiled failed");
    return DDIT_E_TMA;
  }
  fp->p.Lq = a->Lq;
  fp->p.Lk = a->Lk;
  fp->p.q_slot = 0;
  fp->p.k_slot = 0;
  fp->p.v_slot = v_slot;
  fp->p.o_slot = 0;
  fp->p.scale_log2 = a->scale * 1.4426950408889634f;
  fp->p.q_tiles = (a->Lq + fm::BQ - 1) / fm::BQ;
  fp->p.heads = a->heads;
  fp->p.seqs = a->num_seqs;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int units = ((fp->p.q_tiles + 1) / 2) * a->heads * a->num_seqs;
  fp->grid = dim3(units < sms ? units : sms, 1, 1);
  return DDIT_OK;
}

static int fmha_poly() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DDIT_FMHA_POLY");
    v = e ? atoi(e) : 4;
  }
  return v;
}

template <int POLY>
static int fmha_launch_t(const FmhaPlan* fp, cudaStream_t s) {
  static size_t attr[64] = {};
  ensure_smem((const void*)fmha_sm100_kernel<POLY>, fm::SMEM, attr);
  launch_pdl(fmha_sm100_kernel<POLY>, fp->grid, dim3(fm::THREADS), fm::SMEM, s, fp->tmQa, fp->tmQb,
             fp->tmKVa, fp->tmKVb, fp->tmO, fp->p);
  return check_cuda("fmha_sm100_kernel");
}

int fmha_plan_launch(const FmhaPlan* fp, cudaStream_t s) {
  switch (fmha_poly()) {
    case 0: return fmha_launch_t<0>(fp, s);
    case 2: return fmha_launch_t<2>(fp, s);
    case 3: return fmha_launch_t<3>(fp, s);
    default: return fmha_launch_t<4>(fp, s);
  }
}

}  // namespace ddit

#ifdef DDIT_FMHA_TRACE
extern "C" __attribute__((visibility("default"))) int ddit_fmha_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, ddit::g_fm_trace,
                                   sizeof(unsigned long long) * (n < 2048 ? n : 2048));
}
#endif

extern "C" DDIT_API int ddit_attention_tc(const ddit_attn* a, void* stream) {
  ddit::FmhaPlan fp;
  int rc = ddit::fmha_plan_init(&fp, a);
  if (rc) return rc;
  return ddit::fmha_plan_launch(&fp, static_cast<cudaStream_t>(stream));
}
