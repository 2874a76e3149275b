// Implicit-GEMM convolution on tcgen05 for the VAE decoder.
//
// Activations are channels-last bf16 [B][T][H][W][C] (T = 1 for the 2-D spatial decoder).
// One output tile = 128 pixels (R rows x Wt columns of one frame) x BN output channels.
// The K loop runs over (tap, 64-channel block): for tap (dt, dy, dx) the producer TMA-loads
// the input box {64 ch, Wt, R, 1, 1} at (c0, x0+dx-pw, y0+dy-ph, t+dt-pt, b) through a 5-D
// tensor map -- coordinates outside the tensor are zero-filled, which IS the zero padding of
// the convolution (spatial "same" padding and the causal front padding in time of
// CausalConv3d). Weights are [Cout][taps][Cin] (K-major). Accumulation in TMEM (double
// buffered), warp-specialised pipeline as in gemm_sm100.cu; the epilogue adds the bias and an
// optional bf16 residual (TMA-loaded, prefetched one sub-tile ahead) and leaves through
// swizzled smem + TMA stores clipped at the frame edges.
//
// conv2_kernel: the same as a cta_group::2 pair (one TPC): CTA r of the cluster takes pixel tile
// 2 q + r of channel block n, holds half of the BN weight rows, and the leader issues M = 256
// MMAs. Per CTA and k-block the shared memory then sees A (16 KB) + B / 2 written and read instead
// of A + B: at BN = 256 that is 125 instead of 187 B/clk of the 128 B/clk the SM's shared memory
// moves, the bound the 1-CTA kernel sat at.
#include "common.cuh"
#include "cta_pair.cuh"
#include "ddit.h"
#include "capi_internal.h"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>

namespace ddit {
namespace conv {

constexpr int BM = 128, BK = 64, THREADS = 256, TMEM_COLS = 512, ACC_STRIDE = 256;

template <int BN, bool RES>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int EPI = 2 * 16384;  // staging (64 bf16 channels x 128 rows, SW128) x 2
  static constexpr int BAR = 256;
  static constexpr int GNR = 1024;  // GroupNorm statistics: per-warp channel-pair sums [4][8][4][2] fp32
  static constexpr int STAGES_RAW = (232448 - 1024 - BAR - GNR - EPI) / STAGE;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int SMEM = 1024 + STAGES * STAGE + EPI + BAR + GNR;
};

template <int BN, bool RES>
struct Cfg2 {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int EPI = 2 * 16384;
  static constexpr int BAR = 256;
  static constexpr int GNR = 1024;
  static constexpr int STAGES_RAW = (232448 - 1024 - BAR - GNR - EPI) / STAGE;
  static constexpr int STAGES = STAGES_RAW > 10 ? 10 : STAGES_RAW;
  static constexpr int SMEM = 1024 + STAGES * STAGE + EPI + BAR + GNR;
  static_assert(B_BYTES % 1024 == 0, "B half-tile must keep 1024 B swizzle-atom alignment");
};

struct Params {
  int B, T, H, W, Cin, Cout;
  int kt, kh, kw, pt, ph, pw;
  int Wt, R, x_tiles, y_tiles, n_tiles, num_tiles;
  int cblocks, k_blocks;
  int a_bytes;
  int pix_tiles, pair_tiles;  // 2-CTA: pixel tiles, and (pixel-tile pair, channel block) tiles
  const float* bias;
  // optional per-frame GroupNorm statistics of the output: (sum, sum of squares) of group g over
  // the in-frame pixels of pixel tile `slot` of frame n = b T + t -> gn_part[(n G + g) nblk + slot],
  // nblk = x_tiles * y_tiles (the partials gn_finalize_kernel reduces)
  float2* gn_part;
  int gn_G, gn_cg;
  int gn_per_sample;  // 1: statistics per sample b over all T frames, slot = (t y_tiles + yt) x_tiles + xt
};

DDIT_DEV void tma_load_5d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                          int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(c4)
      : "memory");
}
DDIT_DEV void tma_store_5d(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3,
                           int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(m)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
DDIT_DEV void ld32(uint32_t taddr, uint32_t* r) {
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
DDIT_DEV uint32_t sw128(int r, int j) { return (uint32_t)(r * 128 + ((j ^ (r & 7)) << 4)); }
DDIT_DEV void sts4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w)
               : "memory");
}
DDIT_DEV uint4 lds4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}

struct TileCoord {
  int b, t, y0, x0, n0;
};
DDIT_DEV TileCoord decode(const Params& p, int tile, int BN) {
  TileCoord c;
  const int nt = tile % p.n_tiles;
  int pix = tile / p.n_tiles;
  const int xt = pix % p.x_tiles;
  pix /= p.x_tiles;
  const int yt = pix % p.y_tiles;
  pix /= p.y_tiles;
  c.t = pix % p.T;
  c.b = pix / p.T;
  c.y0 = yt * p.R;
  c.x0 = xt * p.Wt;
  c.n0 = nt * BN;
  return c;
}

// GroupNorm statistics of the staged 128 x 64 bf16 output sub-tiles (channels col0 .. col0 + 63,
// rows = the tile's pixels, SW128 rows of 128 B). add(): thread t sums 16 B chunk t % 8 of rows
// 8 (t / 8) .. + 7 (in-frame pixels only, `mask`) per channel pair, a fixed xor tree joins the
// warp's four row sets and lanes 0-7 leave the warp's sums in `red`; flush() -- after the
// epilogue's next named barrier, so no barrier of its own -- joins the four warps in warp order
// and stores one (sum, sum of squares) per group: a deterministic reduction, the same in the
// 1-CTA and the CTA-pair kernel. One `red` suffices: the epilogue has two barriers per sub-tile,
// flush() reads before the second, the next add() writes after it.
DDIT_DEV int gn_nblk(const Params& p) { return p.x_tiles * p.y_tiles * (p.gn_per_sample ? p.T : 1); }

struct GnStats {
  int mask = 0;        // this thread's 8 rows that are in-frame pixels of the current tile
  bool pending = false;
  size_t pidx = 0;     // gn_part index of group col0 / cg of the pending sub-tile
  bool preal = false;

  DDIT_DEV void tile(const Params& p, const TileCoord& tc, int rit) {
    mask = 0;
    const int npix = p.Wt * p.R;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = (rit >> 3) * 8 + i;
      const int yy = tc.y0 + r / p.Wt, xx = tc.x0 + r % p.Wt;
      if (r < npix && yy < p.H && xx < p.W) mask |= 1 << i;
    }
  }
  DDIT_DEV void add(const Params& p, uint32_t sbase, float* red, int rit, const TileCoord& tc,
                    int col0, bool real) {
    const int j = rit & 7, rs = rit >> 3;
    float sm[4] = {0.f, 0.f, 0.f, 0.f}, sq[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (mask >> i & 1) {
        const uint4 q = lds4(sbase + sw128(rs * 8 + i, j));
        const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 a = unpack_bf16(w4[k]);
          sm[k] += a.x + a.y;
          sq[k] = fmaf(a.x, a.x, fmaf(a.y, a.y, sq[k]));
        }
      }
    }
    // the staging buffer's next writer may be a TMA load (residual of a later sub-tile)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
    for (int o = 8; o <= 16; o <<= 1)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        sm[k] += __shfl_xor_sync(0xffffffffu, sm[k], o);
        sq[k] += __shfl_xor_sync(0xffffffffu, sq[k], o);
      }
    if ((rit & 31) < 8) {
      float* w = red + ((rit >> 5) * 8 + j) * 8;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        w[2 * k] = sm[k];
        w[2 * k + 1] = sq[k];
      }
    }
    pending = true;
    preal = real;
    const int slot = (tc.y0 / p.R) * p.x_tiles + tc.x0 / p.Wt;
    if (p.gn_per_sample)
      pidx = ((size_t)tc.b * p.gn_G + col0 / p.gn_cg) * gn_nblk(p) + (size_t)tc.t * p.x_tiles * p.y_tiles + slot;
    else
      pidx = ((size_t)(tc.b * p.T + tc.t) * p.gn_G + col0 / p.gn_cg) * gn_nblk(p) + slot;
  }
  // call after a barrier of all 128 epilogue threads that follows add()
  DDIT_DEV void flush(const Params& p, const float* red, int rit) {
    if (!pending) return;
    pending = false;
    const int pairs = p.gn_cg / 2, ngrp = 64 / p.gn_cg;
    if (rit >= ngrp || !preal) return;
    const float* rb = red;
    float s = 0.f, q = 0.f;
    for (int h = rit * pairs; h < (rit + 1) * pairs; ++h)  // channel pair h = chunk h / 4, k = h % 4
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        s += rb[(w * 8 + (h >> 2)) * 8 + 2 * (h & 3)];
        q += rb[(w * 8 + (h >> 2)) * 8 + 2 * (h & 3) + 1];
      }
    p.gn_part[pidx + (size_t)rit * gn_nblk(p)] = make_float2(s, q);
  }
};

// pair tile pt, CTA rank r -> pixel tile 2 (pt / n_tiles) + r, channel block pt % n_tiles. A rank
// without a pixel tile (odd count) gets the last tile moved past the right edge: its loads are all
// zero fill and it stores nothing (returns false).
DDIT_DEV bool decode2(const Params& p, int pt, int rank, int BN, TileCoord& c) {
  const int nt = pt % p.n_tiles;
  const int pix2 = 2 * (pt / p.n_tiles) + rank;
  const bool real = pix2 < p.pix_tiles;
  int pix = real ? pix2 : p.pix_tiles - 1;
  const int xt = pix % p.x_tiles;
  pix /= p.x_tiles;
  const int yt = pix % p.y_tiles;
  pix /= p.y_tiles;
  c.t = pix % p.T;
  c.b = pix / p.T;
  c.y0 = yt * p.R;
  c.x0 = real ? xt * p.Wt : p.W;
  c.n0 = nt * BN;
  return real;
}

template <int BN, bool RES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    conv2_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                 const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmR,
                 const __grid_constant__ Params p) {
  using C = Cfg2<BN, RES>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint8_t* sE = smem + STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sE + C::EPI);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 2);
  float* gnred = reinterpret_cast<float*>(sE + C::EPI + C::BAR);
  const int warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmY);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);  // 4 epilogue warps x 2 CTAs (the leader's copy is used)
      mbar_init(&rbar[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------------- producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int pt = cid; pt < p.pair_tiles; pt += ncl) {
        TileCoord tc;
        decode2(p, pt, (int)rank, BN, tc);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          const int tap = kb / p.cblocks, cb = kb % p.cblocks;
          const int dx = tap % p.kw, dy = (tap / p.kw) % p.kh, dt = tap / (p.kw * p.kh);
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (p.a_bytes + C::B_BYTES));
          const uint32_t bar0 = cluster_addr(&full[stage], 0);
          tma_load_5d_cg2(sA + stage * C::A_BYTES, &tmX, bar0, cb * BK, tc.x0 + dx - p.pw,
                          tc.y0 + dy - p.ph, tc.t + dt - p.pt, tc.b);
          tma_load_2d_cg2_nohint(sB + stage * C::B_BYTES, &tmW, bar0, kb * BK, tc.n0 + (int)rank * (BN / 2));
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {  // ------------------------------------------ MMA (leader CTA)
    if (rank == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(2 * BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int pt = cid; pt < p.pair_tiles; pt += ncl) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * ACC_STRIDE;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a = smem_u32(sA + stage * C::A_BYTES), b = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16_ss_cg2(d, make_sdesc_sw128(a + 32 * k), make_sdesc_sw128(b + 32 * k), idesc,
                               (kb | k) != 0);
            umma_commit_cg2_mc(&empty[stage]);
            if (kb == p.k_blocks - 1) umma_commit_cg2_mc(&tfull[acc]);
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
    }
  } else if (warp >= 4) {  // ------------------------------------------ epilogue (both CTAs)
    const int ew = warp - 4;
    const int rit = ew * 32 + lane;
    const bool elected = ew == 0 && lane == 0;
    constexpr int NS = BN / 64;
    int acc = 0, cnt = 0;
    uint32_t acc_phase = 0;
    if (RES && elected && cid < p.pair_tiles) {
      TileCoord c0;
      decode2(p, cid, (int)rank, BN, c0);
      mbar_arrive_expect_tx(&rbar[0], p.a_bytes);
      tma_load_5d(sE, &tmR, &rbar[0], c0.n0, c0.x0, c0.y0, c0.t, c0.b);
    }
    const bool gn = p.gn_part != nullptr;
    GnStats gs;
    for (int pt = cid; pt < p.pair_tiles; pt += ncl) {
      TileCoord tc;
      const bool real = decode2(p, pt, (int)rank, BN, tc);
      if (gn) gs.tile(p, tc, rit);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * ACC_STRIDE;
      const uint32_t tcl = cluster_addr(&tempty[acc], 0);
#pragma unroll 1
      for (int sub = 0; sub < NS; ++sub) {
        const int buf = cnt & 1;
        uint8_t* sb = sE + buf * 16384;
        const uint32_t sbase = smem_u32(sb);
        // residual of the next sub-tile into the other buffer; with GroupNorm statistics that
        // buffer may still be read by add() of the previous sub-tile: issue after the barrier
        auto next_res = [&]() {
          const int npt = sub + 1 < NS ? pt : pt + ncl;
          if (npt < p.pair_tiles) {
            TileCoord c1 = tc;
            if (sub + 1 >= NS) decode2(p, npt, (int)rank, BN, c1);
            const int nsub = sub + 1 < NS ? sub + 1 : 0;
            mbar_arrive_expect_tx(&rbar[buf ^ 1], p.a_bytes);
            tma_load_5d(sE + (buf ^ 1) * 16384, &tmR, &rbar[buf ^ 1], c1.n0 + nsub * 64, c1.x0,
                        c1.y0, c1.t, c1.b);
          }
        };
        if (elected) {
          if (RES) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            if (!gn) next_res();
          } else {
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (gn) {
          if (RES && elected) next_res();
          gs.flush(p, gnred, rit);
        }
        if (RES) mbar_wait(&rbar[buf], (cnt >> 1) & 1);
        uint32_t r[64];
        ld32(taddr + sub * 64, r);
        ld32(taddr + sub * 64 + 32, r + 32);
        tmem_ld_wait();
        if (sub == NS - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 31) mbar_arrive_cl_relaxed(tcl);
        }
        const int col0 = tc.n0 + sub * 64;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[8 * j + e]);
          if (p.bias) {
            const float4 b0 = __ldg(reinterpret_cast<const float4*>(p.bias + col0 + 8 * j));
            const float4 b1 = __ldg(reinterpret_cast<const float4*>(p.bias + col0 + 8 * j) + 1);
            v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
            v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
          }
          const uint32_t a = sbase + sw128(rit, j);
          if (RES) {
            const uint4 q = lds4(a);
            const float2 f0 = unpack_bf16(q.x), f1 = unpack_bf16(q.y), f2 = unpack_bf16(q.z),
                         f3 = unpack_bf16(q.w);
            v[0] += f0.x; v[1] += f0.y; v[2] += f1.x; v[3] += f1.y;
            v[4] += f2.x; v[5] += f2.y; v[6] += f3.x; v[7] += f3.y;
          }
          sts4(a, pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
               pack_bf16(v[6], v[7]));
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (elected && real) {
          tma_store_5d(&tmY, sb, col0, tc.x0, tc.y0, tc.t, tc.b);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (gn) gs.add(p, sbase, gnred, rit, tc, col0, real);
        ++cnt;
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (gn) {
      asm volatile("bar.sync 1, 128;" ::: "memory");
      gs.flush(p, gnred, rit);
    }
    if (elected) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(TMEM_COLS)
                 : "memory");
  }
}

template <int BN, bool RES>
__global__ void __launch_bounds__(THREADS, 1)
    conv_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmR,
                const __grid_constant__ Params p) {
  using C = Cfg<BN, RES>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint8_t* sE = smem + STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sE + C::EPI);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 2);
  float* gnred = reinterpret_cast<float*>(sE + C::EPI + C::BAR);
  const int warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmY);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
      mbar_init(&rbar[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------------- producer
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        const TileCoord tc = decode(p, tile, BN);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          const int tap = kb / p.cblocks, cb = kb % p.cblocks;
          const int dx = tap % p.kw, dy = (tap / p.kw) % p.kh, dt = tap / (p.kw * p.kh);
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], p.a_bytes + C::B_BYTES);
          tma_load_5d(sA + stage * C::A_BYTES, &tmX, &full[stage], cb * BK, tc.x0 + dx - p.pw,
                      tc.y0 + dy - p.ph, tc.t + dt - p.pt, tc.b);
          tma_load_2d(sB + stage * C::B_BYTES, &tmW, &full[stage], kb * BK, tc.n0);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {  // ------------------------------------------ MMA
    constexpr uint32_t idesc = make_idesc_bf16(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + acc * ACC_STRIDE;
      for (int kb = 0; kb < p.k_blocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a = smem_u32(sA + stage * C::A_BYTES), b = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16_ss(d, make_sdesc_sw128(a + 32 * k), make_sdesc_sw128(b + 32 * k), idesc,
                         (kb | k) != 0);
          umma_commit(&empty[stage]);
          if (kb == p.k_blocks - 1) umma_commit(&tfull[acc]);
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
  } else if (warp >= 4) {  // ------------------------------------------ epilogue
    const int ew = warp - 4;
    const int rit = ew * 32 + lane;
    const bool elected = ew == 0 && lane == 0;
    constexpr int NS = BN / 64;
    int acc = 0, cnt = 0;
    uint32_t acc_phase = 0;
    if (RES && elected && (int)blockIdx.x < p.num_tiles) {
      const TileCoord c0 = decode(p, blockIdx.x, BN);
      mbar_arrive_expect_tx(&rbar[0], p.a_bytes);
      tma_load_5d(sE, &tmR, &rbar[0], c0.n0, c0.x0, c0.y0, c0.t, c0.b);
    }
    const bool gn = p.gn_part != nullptr;
    GnStats gs;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      const TileCoord tc = decode(p, tile, BN);
      if (gn) gs.tile(p, tc, rit);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * ACC_STRIDE;
#pragma unroll 1
      for (int sub = 0; sub < NS; ++sub) {
        const int buf = cnt & 1;
        uint8_t* sb = sE + buf * 16384;
        const uint32_t sbase = smem_u32(sb);
        auto next_res = [&]() {  // see conv2_kernel
          const int nt = sub + 1 < NS ? tile : tile + (int)gridDim.x;
          if (nt < p.num_tiles) {
            const TileCoord c1 = sub + 1 < NS ? tc : decode(p, nt, BN);
            const int nsub = sub + 1 < NS ? sub + 1 : 0;
            mbar_arrive_expect_tx(&rbar[buf ^ 1], p.a_bytes);
            tma_load_5d(sE + (buf ^ 1) * 16384, &tmR, &rbar[buf ^ 1], c1.n0 + nsub * 64, c1.x0,
                        c1.y0, c1.t, c1.b);
          }
        };
        if (elected) {
          if (RES) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            if (!gn) next_res();
          } else {
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (gn) {
          if (RES && elected) next_res();
          gs.flush(p, gnred, rit);
        }
        if (RES) mbar_wait(&rbar[buf], (cnt >> 1) & 1);
        uint32_t r[64];
        ld32(taddr + sub * 64, r);
        ld32(taddr + sub * 64 + 32, r + 32);
        tmem_ld_wait();
        if (sub == NS - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 31) mbar_arrive_relaxed(&tempty[acc]);
        }
        const int col0 = tc.n0 + sub * 64;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[8 * j + e]);
          if (p.bias) {
            const float4 b0 = __ldg(reinterpret_cast<const float4*>(p.bias + col0 + 8 * j));
            const float4 b1 = __ldg(reinterpret_cast<const float4*>(p.bias + col0 + 8 * j) + 1);
            v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
            v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
          }
          const uint32_t a = sbase + sw128(rit, j);
          if (RES) {
            const uint4 q = lds4(a);
            const float2 f0 = unpack_bf16(q.x), f1 = unpack_bf16(q.y), f2 = unpack_bf16(q.z),
                         f3 = unpack_bf16(q.w);
            v[0] += f0.x; v[1] += f0.y; v[2] += f1.x; v[3] += f1.y;
            v[4] += f2.x; v[5] += f2.y; v[6] += f3.x; v[7] += f3.y;
          }
          sts4(a, pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
               pack_bf16(v[6], v[7]));
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (elected) {
          tma_store_5d(&tmY, sb, col0, tc.x0, tc.y0, tc.t, tc.b);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (gn) gs.add(p, sbase, gnred, rit, tc, col0, true);
        ++cnt;
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (gn) {
      asm volatile("bar.sync 1, 128;" ::: "memory");
      gs.flush(p, gnred, rit);
    }
    if (elected) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem_base);
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

// channels-last [B][T][H][W][C] bf16, box {64, Wt, R, 1, 1}, 128 B swizzle
static bool map_act(CUtensorMap* m, const void* base, int B, int T, int H, int W, int C, int Wt,
                    int R) {
  cuuint64_t dims[5] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)T, (cuuint64_t)B};
  cuuint64_t st[4] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2,
                      (cuuint64_t)T * H * W * C * 2};
  cuuint32_t box[5] = {64, (cuuint32_t)Wt, (cuuint32_t)R, 1, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return encoder()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, st, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <int BN, bool RES>
static int launch(const CUtensorMap& x, const CUtensorMap& w, const CUtensorMap& y,
                  const CUtensorMap& r, const Params& p, int grid, bool pair, cudaStream_t s) {
  if (pair) {
    using C = Cfg2<BN, RES>;
    static size_t attr2[64] = {};
    ensure_smem((const void*)conv2_kernel<BN, RES>, C::SMEM, attr2);
    conv2_kernel<BN, RES><<<grid, THREADS, C::SMEM, s>>>(x, w, y, r, p);
    return check_cuda("conv2_kernel");
  }
  using C = Cfg<BN, RES>;
  static size_t attr[64] = {};
  ensure_smem((const void*)conv_kernel<BN, RES>, C::SMEM, attr);
  conv_kernel<BN, RES><<<grid, THREADS, C::SMEM, s>>>(x, w, y, r, p);
  return check_cuda("conv_kernel");
}

static int g_conv_tiles = -1;  // DDIT_CONV_TILES=0: 128-pixel rows (W >= 128) / whole rows
static bool conv_tile_search_enabled() {
  if (g_conv_tiles < 0) {
    const char* e = getenv("DDIT_CONV_TILES");
    g_conv_tiles = (e && e[0] == '0') ? 0 : 1;
  }
  return g_conv_tiles != 0;
}

static int g_conv_pair = -1;  // DDIT_CONV_2CTA=0: 1-CTA tiles only
static bool conv_pair_enabled() {
  if (g_conv_pair < 0) {
    const char* e = getenv("DDIT_CONV_2CTA");
    g_conv_pair = (e && e[0] == '0') ? 0 : 1;
  }
  return g_conv_pair != 0;
}

// pixel tile = R rows x Wt columns (Wt * R <= 128, the MMA's M): the shape with the fewest tiles
// per frame, i.e. the least MMA work on pixels past the frame edge (e.g. W = 432: 16 x 8 tiles,
// 810 per 240-row frame, instead of 128 x 1, 960); ties keep the wider rows. Results do not
// depend on the tiling (same K order per pixel).
static void pixel_tile(int H, int W, int* Wt, int* R) {
  auto tiles_of = [&](int wt, int r) { return (long)((W + wt - 1) / wt) * ((H + r - 1) / r); };
  int bw = W < 128 ? W : 128;
  int br = std::max(1, std::min(H, 128 / bw));
  if (conv_tile_search_enabled()) {
    for (int wt : {128, 64, 32, 16}) {
      if (wt > W) continue;
      const int r = std::max(1, std::min(H, 128 / wt));
      if (tiles_of(wt, r) < tiles_of(bw, br)) {
        bw = wt;
        br = r;
      }
    }
  }
  *Wt = bw;
  *R = br;
}

}  // namespace conv
}  // namespace ddit

using namespace ddit;

extern "C" DDIT_API int ddit_set_conv_tile_search(int on) {
  conv::g_conv_tiles = on ? 1 : 0;
  return DDIT_OK;
}

extern "C" DDIT_API int ddit_set_conv_2cta(int on) {
  conv::g_conv_pair = on ? 1 : 0;
  return DDIT_OK;
}

extern "C" DDIT_API int ddit_conv_frame_tiles(int H, int W) {
  if (H < 1 || W < 1) return 0;
  int wt = 0, r = 0;
  conv::pixel_tile(H, W, &wt, &r);
  return ((W + wt - 1) / wt) * ((H + r - 1) / r);
}

extern "C" DDIT_API int ddit_conv(const ddit_conv_args* a, void* stream) {
  using namespace conv;
  if (!encoder()) {
    set_error("conv: cuTensorMapEncodeTiled unavailable");
    return DDIT_E_TMA;
  }
  if (a->Cin % 64 || a->Cout % 64 || a->B < 1 || a->T < 1 || a->H < 1 || a->W < 1) {
    set_error("conv: Cin and Cout must be multiples of 64 (got %d, %d)", a->Cin, a->Cout);
    return DDIT_E_INVALID;
  }
  const int bn = a->Cout % 256 == 0 ? 256 : (a->Cout % 128 == 0 ? 128 : 64);
  Params p;
  memset(&p, 0, sizeof p);
  p.B = a->B; p.T = a->T; p.H = a->H; p.W = a->W; p.Cin = a->Cin; p.Cout = a->Cout;
  p.kt = a->kt; p.kh = a->kh; p.kw = a->kw;
  p.pt = a->causal_time ? a->kt - 1 : a->kt / 2;
  p.ph = a->kh / 2;
  p.pw = a->kw / 2;
  pixel_tile(a->H, a->W, &p.Wt, &p.R);
  p.x_tiles = (a->W + p.Wt - 1) / p.Wt;
  p.y_tiles = (a->H + p.R - 1) / p.R;
  p.n_tiles = a->Cout / bn;
  p.num_tiles = a->B * a->T * p.y_tiles * p.x_tiles * p.n_tiles;
  p.cblocks = a->Cin / 64;
  p.k_blocks = a->kt * a->kh * a->kw * p.cblocks;
  p.a_bytes = p.Wt * p.R * 128;
  p.pix_tiles = a->B * a->T * p.y_tiles * p.x_tiles;
  p.pair_tiles = ((p.pix_tiles + 1) / 2) * p.n_tiles;
  p.bias = a->bias;
  if (a->gn_part) {
    const int G = a->gn_groups;
    if (G < 1 || a->Cout % G || (a->Cout / G) % 2 || 64 % (a->Cout / G)) {
      set_error("conv: GroupNorm statistics need Cout / groups in {2, 4, ..., 64} (Cout %d, groups %d)",
                a->Cout, G);
      return DDIT_E_INVALID;
    }
    p.gn_part = reinterpret_cast<float2*>(a->gn_part);
    p.gn_G = G;
    p.gn_cg = a->Cout / G;
    p.gn_per_sample = a->gn_per_sample ? 1 : 0;
  }
  CUtensorMap tx, tw, ty, tr;
  memset(&tr, 0, sizeof tr);
  bool ok = map_act(&tx, a->x, a->B, a->T, a->H, a->W, a->Cin, p.Wt, p.R) &&
            map_act(&ty, a->y, a->B, a->T, a->H, a->W, a->Cout, p.Wt, p.R);
  if (ok && a->residual) ok = map_act(&tr, a->residual, a->B, a->T, a->H, a->W, a->Cout, p.Wt, p.R);
  {
    const int K = p.k_blocks * 64;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)a->Cout};
    cuuint64_t st[1] = {(cuuint64_t)K * 2};
    // CTA pairs load half the weight rows each
    const bool pair = conv_pair_enabled() && p.pair_tiles >= num_sms() / 2;
    cuuint32_t box[2] = {64, (cuuint32_t)(pair ? bn / 2 : bn)};
    cuuint32_t es[2] = {1, 1};
    ok = ok && encoder()(&tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a->w), dims, st,
                         box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  if (!ok) {
    set_error("conv: tensor map encoding failed");
    return DDIT_E_TMA;
  }
  if (!a->residual) tr = ty;
  const bool pair = conv_pair_enabled() && p.pair_tiles >= num_sms() / 2;
  const int grid = pair ? 2 * (p.pair_tiles < num_sms() / 2 ? p.pair_tiles : num_sms() / 2)
                        : (p.num_tiles < num_sms() ? p.num_tiles : num_sms());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool res = a->residual != nullptr;
  switch (bn) {
    case 256: return res ? launch<256, true>(tx, tw, ty, tr, p, grid, pair, s) : launch<256, false>(tx, tw, ty, tr, p, grid, pair, s);
    case 128: return res ? launch<128, true>(tx, tw, ty, tr, p, grid, pair, s) : launch<128, false>(tx, tw, ty, tr, p, grid, pair, s);
    default: return res ? launch<64, true>(tx, tw, ty, tr, p, grid, pair, s) : launch<64, false>(tx, tw, ty, tr, p, grid, pair, s);
  }
}
