// Persistent warp-specialised tcgen05 GEMM for sm_100a with the STDiT epilogues fused.
//
//   warp 0      : TMA producer (one elected lane) -- A/B k-blocks into a STAGES-deep smem ring
//   warp 1      : MMA issuer   (one elected lane) -- tcgen05.mma 128xBNx16 into TMEM
//   warp 2      : TMEM allocator (512 columns: two accumulator buffers at columns 0 / 256)
//   warps 4..7  : epilogue -- tcgen05.ld (one accumulator row per thread) -> fused op -> global
//
// The accumulator is double-buffered in TMEM so the epilogue of tile i overlaps the MMAs of
// tile i+1. Tiles are distributed round-robin over a grid of min(#tiles, #SMs) CTAs.
// Shapes in the DDiT step: M = tokens (ragged, TMA zero-fills the
// tail, and the K tail), K in {1152, 4096, 4608}, N in {1152, 2304, 3456, 4608}; N % BN == 0.
#include "common.cuh"
#include "gemm_sm100.cuh"

#include <cstdio>
#include <cstring>
#include <mutex>

namespace ddit {

static constexpr int BM = 128;
static constexpr int BK = 64;
static constexpr int kThreads = 256;
static constexpr int kTmemCols = 512;
static constexpr int kAccStride = 256;  // TMEM column offset of accumulator buffer 1

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (212 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int BAR_BYTES = 256;
  static constexpr int SMEM = 1024 /*align slack*/ + STAGES * STAGE_BYTES + BAR_BYTES;
  static_assert(B_BYTES % 1024 == 0, "B tile must keep 1024 B swizzle-atom alignment");
  static_assert(BN % 16 == 0 && BN <= 256, "invalid UMMA N");
};

DDIT_DEV void tmem_ld_32x32b_x8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

// ------------------------------------------------------------------ epilogues
template <int BN, int EPI>
DDIT_DEV void epilogue_generic(const EpiParams& ep, uint32_t taddr, int row, int M, int n0) {
  const bool live = row < M;
#pragma unroll 1
  for (int c = 0; c < BN; c += 16) {
    uint32_t r[16];
    tmem_ld_32x32b_x16(taddr + c, r);
    tmem_ld_wait();
    if (!live) continue;
    const int col = n0 + c;
    float v[16];
    if (ep.bias) {
      const float4* b4 = reinterpret_cast<const float4*>(ep.bias + col);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float4 b = __ldg(b4 + q);
        v[4 * q + 0] = __uint_as_float(r[4 * q + 0]) + b.x;
        v[4 * q + 1] = __uint_as_float(r[4 * q + 1]) + b.y;
        v[4 * q + 2] = __uint_as_float(r[4 * q + 2]) + b.z;
        v[4 * q + 3] = __uint_as_float(r[4 * q + 3]) + b.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = __uint_as_float(r[e]);
    }
    if constexpr (EPI == EPI_BF16 || EPI == EPI_GELU_BF16) {
      if constexpr (EPI == EPI_GELU_BF16) {
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = gelu_tanh(v[e]);
      }
      uint4* o = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) +
                                          (size_t)row * ep.ldo + col);
      o[0] = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                        pack_bf16(v[6], v[7]));
      o[1] = make_uint4(pack_bf16(v[8], v[9]), pack_bf16(v[10], v[11]), pack_bf16(v[12], v[13]),
                        pack_bf16(v[14], v[15]));
    } else if constexpr (EPI == EPI_F32) {
      float4* o = reinterpret_cast<float4*>(static_cast<float*>(ep.out) + (size_t)row * ep.ldo + col);
#pragma unroll
      for (int q = 0; q < 4; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else if constexpr (EPI == EPI_RESID) {
      float4* rp = reinterpret_cast<float4*>(ep.resid + (size_t)row * ep.ldr + col);
      float g[16];
      if (ep.gate) {
        const float4* g4 =
            reinterpret_cast<const float4*>(ep.gate + (size_t)(row / ep.rows_per_b) * ep.gate_stride + col);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float4 t = __ldg(g4 + q);
          g[4 * q] = t.x; g[4 * q + 1] = t.y; g[4 * q + 2] = t.z; g[4 * q + 3] = t.w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) g[e] = 1.0f;
      }
      float nv[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float4 x = rp[q];
        nv[4 * q + 0] = x.x + g[4 * q + 0] * v[4 * q + 0];
        nv[4 * q + 1] = x.y + g[4 * q + 1] * v[4 * q + 1];
        nv[4 * q + 2] = x.z + g[4 * q + 2] * v[4 * q + 2];
        nv[4 * q + 3] = x.w + g[4 * q + 3] * v[4 * q + 3];
        rp[q] = make_float4(nv[4 * q], nv[4 * q + 1], nv[4 * q + 2], nv[4 * q + 3]);
      }
      if (ep.out2) {
        uint4* o = reinterpret_cast<uint4*>(ep.out2 + (size_t)row * ep.ldo2 + col);
        o[0] = make_uint4(pack_bf16(nv[0], nv[1]), pack_bf16(nv[2], nv[3]), pack_bf16(nv[4], nv[5]),
                          pack_bf16(nv[6], nv[7]));
        o[1] = make_uint4(pack_bf16(nv[8], nv[9]), pack_bf16(nv[10], nv[11]),
                          pack_bf16(nv[12], nv[13]), pack_bf16(nv[14], nv[15]));
      }
    }
  }
}

// QKV epilogue: the 144-column tile holds two whole heads (head_dim 72) of one of q/k/v.
// q,k: bias -> per-head RMSNorm (weight) -> optional interleaved RoPE by frame index.
DDIT_DEV void epilogue_qkv(const EpiParams& ep, uint32_t taddr, int row, int M, int n0) {
  constexpr int HD = 72;
  const bool live = row < M;
  const int section = n0 / ep.hidden;  // 0 q, 1 k, 2 v
  __nv_bfloat16* out = static_cast<__nv_bfloat16*>(ep.out) + (size_t)row * ep.ldo;
  int pos = 0;
  if (ep.rope) pos = (row / ep.rope_S) % ep.rope_T;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    const int c0 = h * HD;
    if (section < 2) {
      float ss = 0.f;
#pragma unroll 1
      for (int j = 0; j < HD / 8; ++j) {
        uint32_t r[8];
        tmem_ld_32x32b_x8(taddr + c0 + j * 8, r);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float v = __uint_as_float(r[e]) + __ldg(ep.bias + n0 + c0 + j * 8 + e);
          ss += v * v;
        }
      }
      const float inv = rsqrtf(ss * (1.0f / HD) + ep.eps);
      const float* w = section == 0 ? ep.qnorm_w : ep.knorm_w;
#pragma unroll 1
      for (int j = 0; j < HD / 8; ++j) {
        uint32_t r[8];
        tmem_ld_32x32b_x8(taddr + c0 + j * 8, r);
        tmem_ld_wait();
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          v[e] = (__uint_as_float(r[e]) + __ldg(ep.bias + n0 + c0 + j * 8 + e)) * inv *
                 __ldg(w + j * 8 + e);
        if (ep.rope) {
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            float2 cs = __ldg(ep.rope_tab + pos * (HD / 2) + (j * 8 + e) / 2);
            float a = v[e], b = v[e + 1];
            v[e] = a * cs.x - b * cs.y;
            v[e + 1] = b * cs.x + a * cs.y;
          }
        }
        if (live)
          *reinterpret_cast<uint4*>(out + n0 + c0 + j * 8) =
              make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                         pack_bf16(v[6], v[7]));
      }
    } else {
#pragma unroll 1
      for (int j = 0; j < HD / 8; ++j) {
        uint32_t r[8];
        tmem_ld_32x32b_x8(taddr + c0 + j * 8, r);
        tmem_ld_wait();
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          v[e] = __uint_as_float(r[e]) + __ldg(ep.bias + n0 + c0 + j * 8 + e);
        if (live)
          *reinterpret_cast<uint4*>(out + n0 + c0 + j * 8) =
              make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                         pack_bf16(v[6], v[7]));
      }
    }
  }
}

// ------------------------------------------------------------------ kernel
template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
                        const __grid_constant__ EpiParams ep) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int m_tiles = (M + BM - 1) / BM;
  const int n_tiles = N / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int k_blocks = (K + BK - 1) / BK;  // TMA zero-fills the K tail

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

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
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m_blk = tile / n_tiles;
      const int n_blk = tile % n_tiles;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m_blk * BM + ew * 32 + lane;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * kAccStride;
      if constexpr (EPI == EPI_QKV) {
        epilogue_qkv(ep, taddr, row, M, n_blk * BN);
      } else {
        epilogue_generic<BN, EPI>(ep, taddr, row, M, n_blk * BN);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
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

// 2-D bf16 tensor map over a row-major [rows, cols] matrix with row stride ld (elements),
// box = [box_rows, 64 cols], 128 B swizzle, zero fill out of bounds.
static int make_tmap_bf16(CUtensorMap* m, const void* base, int rows, int cols, int ld,
                          int box_rows) {
  PFN_tmapEncodeTiled enc = get_encode();
  if (!enc) {
    snprintf(g_err, sizeof g_err, "cuTensorMapEncodeTiled unavailable");
    return -1;
  }
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_err, sizeof g_err, "cuTensorMapEncodeTiled failed (%d) rows=%d cols=%d ld=%d",
             (int)r, rows, cols, ld);
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

int gemm_plan_init(GemmPlan* p, const void* A, int lda, const void* B, int ldb, int M, int N,
                   int K, int epi, const EpiParams& ep, int bn) {
  if (bn != 128 && bn != 144 && bn != 192 && bn != 256) {
    snprintf(g_err, sizeof g_err, "unsupported BN %d", bn);
    return -2;
  }
  if (M <= 0 || N % bn != 0 || K <= 0) {
    snprintf(g_err, sizeof g_err, "bad GEMM shape M=%d N=%d K=%d BN=%d", M, N, K, bn);
    return -2;
  }
  if (epi == EPI_QKV && (bn != 144 || ep.hidden % 144 != 0)) {
    snprintf(g_err, sizeof g_err, "EPI_QKV needs BN=144 and hidden %% 144 == 0");
    return -2;
  }
  if ((lda * 2) % 16 || (ldb * 2) % 16 || (reinterpret_cast<uintptr_t>(A) & 15) ||
      (reinterpret_cast<uintptr_t>(B) & 15)) {
    snprintf(g_err, sizeof g_err, "GEMM operands must be 16-byte aligned");
    return -2;
  }
  memset(p, 0, sizeof *p);
  if (make_tmap_bf16(&p->tmA, A, M, K, lda, BM)) return -3;
  if (make_tmap_bf16(&p->tmB, B, N, K, ldb, bn)) return -3;
  p->M = M;
  p->N = N;
  p->K = K;
  p->bn = bn;
  p->epi = epi;
  p->ep = ep;
  const int tiles = ((M + BM - 1) / BM) * (N / bn);
  p->grid = tiles < num_sms() ? tiles : num_sms();
  return 0;
}

template <int BN, int EPI>
static int launch_t(const GemmPlan* p, cudaStream_t s) {
  constexpr int smem = GemmCfg<BN>::SMEM;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN, EPI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) {
      snprintf(g_err, sizeof g_err, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
      return -4;
    }
    attr_set = true;
  }
  gemm_bf16_tn_kernel<BN, EPI><<<p->grid, kThreads, smem, s>>>(p->tmA, p->tmB, p->M, p->N, p->K,
                                                                p->ep);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof g_err, "gemm launch: %s", cudaGetErrorString(e));
    return -4;
  }
  return 0;
}

template <int BN>
static int launch_bn(const GemmPlan* p, cudaStream_t s) {
  switch (p->epi) {
    case EPI_BF16: return launch_t<BN, EPI_BF16>(p, s);
    case EPI_GELU_BF16: return launch_t<BN, EPI_GELU_BF16>(p, s);
    case EPI_RESID: return launch_t<BN, EPI_RESID>(p, s);
    case EPI_F32: return launch_t<BN, EPI_F32>(p, s);
    default: break;
  }
  snprintf(g_err, sizeof g_err, "epilogue %d not instantiated for BN %d", p->epi, BN);
  return -2;
}

int gemm_plan_launch(const GemmPlan* p, cudaStream_t s) {
  if (p->epi == EPI_QKV) return launch_t<144, EPI_QKV>(p, s);
  switch (p->bn) {
    case 128: return launch_bn<128>(p, s);
    case 144: return launch_bn<144>(p, s);
    case 192: return launch_bn<192>(p, s);
    case 256: return launch_bn<256>(p, s);
  }
  return -2;
}

}  // namespace ddit
