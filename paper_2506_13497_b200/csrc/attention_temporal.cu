// Temporal attention for short sequences (T <= 32 frames).
//
// The temporal sequences of the DDiT step are the T frames of one token position: rows
// base + t*tok of the token-major QKV matrix. A token's whole QKV row (3*C bf16 = 6.9 KB at
// XL/2) is contiguous, so one CTA takes one (batch, position) and ALL heads: it streams the T
// full rows into smem with 16 B cp.async (fully coalesced), runs every head's T x T attention
// with bf16 mma.sync from smem (head_dim 72 = 4 k16 + 1 k8 steps: no padding, no foreign
// columns), and writes the T output rows back through smem (over the consumed q columns)
// with coalesced 16 B stores.
// Work is memory-bound (q/k/v read once, o written once): the roofline is HBM bytes.
#include "common.cuh"
#include "ddit.h"
#include "capi_internal.h"

namespace ddit {

static constexpr int TA_THREADS = 256;  // 8 warps; warp w handles heads w, w+8, ...
static constexpr int TA_MAXT = 32;

struct TemporalParams {
  const __nv_bfloat16* qkv;  // row r: [q (C) | k (C) | v (C)], head h at 72h within each
  __nv_bfloat16* o;          // row r: [C]
  int ldqkv, ldo;
  int T, C, heads;
  int inner, outer, tok;     // position i -> base row (i / inner) * outer + (i % inner)
  float scale_log2;
};

DDIT_DEV void cp16(uint32_t smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(g));
}
DDIT_DEV void ldsm4(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(a));
}
DDIT_DEV void ldsm2(uint32_t a, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(a));
}
DDIT_DEV void ldsm2t(uint32_t a, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(a));
}
DDIT_DEV void ldsm4t(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(a));
}
DDIT_DEV void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                       uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
DDIT_DEV void mma1688(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(b0));
}

// One (head, 16-query-row tile) of a T x T problem with T <= 32 (NT = key tiles of 8).
// The output of (h, mt) overwrites the q columns of head h in rows mt*16.. (already in regs).
template <int NT>
DDIT_DEV void temporal_head(__nv_bfloat16* sm, int pitch, int C, int h, int mt, int T,
                            float scale_log2) {
  const int lane = lane_id();
  const int g = lane >> 2, t4 = lane & 3;
  const int qcol = h * 72, kcol = C + h * 72, vcol = 2 * C + h * 72;
  const uint32_t base = smem_u32(sm);
  // Q fragments (rows mt*16 .. +15): 4 k16 steps + 1 k8 step
  uint32_t qa[4][4], qb[2];
  {
    const int r = mt * 16 + (lane & 15);
    const uint32_t a = base + (uint32_t)(r * pitch + qcol + (lane >> 4) * 8) * 2;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) ldsm4(a + ks * 32, qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
    ldsm2(base + (uint32_t)(r * pitch + qcol + 64) * 2, qb[0], qb[1]);
  }
  float s[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
    const int key = n * 8 + (lane & 7);
    const uint32_t a = base + (uint32_t)(key * pitch + kcol + ((lane >> 3) & 1) * 8) * 2;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t b0, b1;
      ldsm2(a + ks * 32, b0, b1);
      mma16816(s[n], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
    }
    uint32_t b0, b1;
    ldsm2(base + (uint32_t)(key * pitch + kcol + 64) * 2, b0, b1);  // lanes 0..7 used
    mma1688(s[n], qb[0], qb[1], b0);
  }
  // softmax over keys < T (rows g and g+8)
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const bool ok = n * 8 + 2 * t4 + e < T;
      s[n][e] = ok ? s[n][e] * scale_log2 : -INFINITY;
      s[n][2 + e] = ok ? s[n][2 + e] * scale_log2 : -INFINITY;
      m0 = fmaxf(m0, s[n][e]);
      m1 = fmaxf(m1, s[n][2 + e]);
    }
  }
  m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
  m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
  m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
  m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
  float l0 = 0.f, l1 = 0.f;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    s[n][0] = exp2f(s[n][0] - m0);
    s[n][1] = exp2f(s[n][1] - m0);
    s[n][2] = exp2f(s[n][2] - m1);
    s[n][3] = exp2f(s[n][3] - m1);
    l0 += s[n][0] + s[n][1];
    l1 += s[n][2] + s[n][3];
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  // O = P V : keys in k16 chunks (NT/2 of them), d in 9 n8 tiles
  float o[9][4];
#pragma unroll
  for (int i = 0; i < 9; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < NT / 2; ++kk) {
    const uint32_t a0 = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
    const uint32_t a1 = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
    const uint32_t a2 = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
    const uint32_t a3 = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
    const int key = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
    for (int dp = 0; dp < 4; ++dp) {
      uint32_t b0, b1, b2, b3;
      ldsm4t(base + (uint32_t)(key * pitch + vcol + dp * 16 + (lane >> 4) * 8) * 2, b0, b1, b2, b3);
      mma16816(o[2 * dp], a0, a1, a2, a3, b0, b1);
      mma16816(o[2 * dp + 1], a0, a1, a2, a3, b2, b3);
    }
    uint32_t b0, b1;
    ldsm2t(base + (uint32_t)(key * pitch + vcol + 64) * 2, b0, b1);
    mma16816(o[8], a0, a1, a2, a3, b0, b1);
  }
  const float i0 = 1.f / l0, i1 = 1.f / l1;
  const int r0 = mt * 16 + g, r1 = r0 + 8;
#pragma unroll
  for (int nt = 0; nt < 9; ++nt) {
    const int d = h * 72 + nt * 8 + 2 * t4;
    if (r0 < T) *reinterpret_cast<uint32_t*>(sm + r0 * pitch + d) = pack_bf16(o[nt][0] * i0, o[nt][1] * i0);
    if (r1 < T) *reinterpret_cast<uint32_t*>(sm + r1 * pitch + d) = pack_bf16(o[nt][2] * i1, o[nt][3] * i1);
  }
}

template <int NT>
__global__ void __launch_bounds__(TA_THREADS)
    temporal_attn_kernel(const __grid_constant__ TemporalParams p) {
  extern __shared__ __align__(16) uint8_t ta_smem[];
  const int pitch = 3 * p.C + 8;  // +16 B: conflict-free ldmatrix rows
  __nv_bfloat16* sm = reinterpret_cast<__nv_bfloat16*>(ta_smem);
  pdl_wait();
  const int pos = blockIdx.x;
  const int base_row = (pos / p.inner) * p.outer + (pos % p.inner);
  const int rows = NT * 8;
  // stream the T qkv rows (zero rows T..rows-1: their P is 0 but V must be finite)
  const int chunks = 3 * p.C / 8;
  const uint32_t sbase = smem_u32(sm);
  for (int c = threadIdx.x; c < rows * chunks; c += TA_THREADS) {
    const int r = c / chunks, ch = c % chunks;
    if (r < p.T)
      cp16(sbase + (uint32_t)(r * pitch + ch * 8) * 2,
           p.qkv + (size_t)(base_row + r * p.tok) * p.ldqkv + ch * 8);
    else
      *reinterpret_cast<uint4*>(sm + r * pitch + ch * 8) = make_uint4(0, 0, 0, 0);
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const int warp = warp_id();
  const int mtiles = (p.T + 15) / 16;
  for (int job = warp; job < p.heads * mtiles; job += TA_THREADS / 32)
    temporal_head<NT>(sm, pitch, p.C, job / mtiles, job % mtiles, p.T, p.scale_log2);
  __syncthreads();
  const int ochunks = p.C / 8;
  for (int c = threadIdx.x; c < p.T * ochunks; c += TA_THREADS) {
    const int r = c / ochunks, ch = c % ochunks;
    *reinterpret_cast<uint4*>(p.o + (size_t)(base_row + r * p.tok) * p.ldo + ch * 8) =
        *reinterpret_cast<const uint4*>(sm + r * pitch + ch * 8);
  }
}

// q/k/v must be the three C-wide sections of one row-major QKV matrix (ld = 3C).
int temporal_attention_launch(const ddit_attn* a, cudaStream_t s) {
  const int C = a->heads * a->head_dim;
  const auto* q = static_cast<const __nv_bfloat16*>(a->q);
  if (a->head_dim != 72 || a->Lq != a->Lk || a->Lq > TA_MAXT || a->ldq != 3 * C ||
      static_cast<const __nv_bfloat16*>(a->k) != q + C ||
      static_cast<const __nv_bfloat16*>(a->v) != q + 2 * C || a->ldk != a->ldq ||
      a->ldv != a->ldq || a->q_inner_stride != 1 || a->kv_tok != a->q_tok ||
      a->kv_outer != a->q_outer || a->kv_inner != a->q_inner) {
    set_error("temporal attention: needs one QKV matrix, T <= 32, shared q/kv index map");
    return DDIT_E_INVALID;
  }
  TemporalParams p;
  p.qkv = q;
  p.o = static_cast<__nv_bfloat16*>(a->o);
  p.ldqkv = a->ldq;
  p.ldo = a->ldo;
  p.T = a->Lq;
  p.C = C;
  p.heads = a->heads;
  p.inner = a->q_inner > 0 ? a->q_inner : 1;
  p.outer = a->q_outer;
  p.tok = a->q_tok;
  p.scale_log2 = a->scale * 1.4426950408889634f;
  const int NT = p.T <= 16 ? 2 : 4;
  const size_t smem = (size_t)NT * 8 * (3 * C + 8) * 2;
  if (smem > 227 * 1024) {
    set_error("temporal attention: T x 4C row block does not fit in shared memory");
    return DDIT_E_INVALID;
  }
  auto kern = NT == 2 ? temporal_attn_kernel<2> : temporal_attn_kernel<4>;
  static size_t attr[2][64] = {};
  ensure_smem((const void*)kern, 227 * 1024, attr[NT == 4]);
  launch_pdl(kern, dim3(a->num_seqs), dim3(TA_THREADS), smem, s, p);
  return check_cuda("temporal_attn_kernel");
}

}  // namespace ddit

extern "C" DDIT_API int ddit_attention_temporal(const ddit_attn* a, void* stream) {
  return ddit::temporal_attention_launch(a, static_cast<cudaStream_t>(stream));
}
