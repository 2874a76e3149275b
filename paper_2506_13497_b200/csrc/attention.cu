// Flash attention for the STDiT3 spatial / temporal / cross attention (head_dim 72).
//
// One CTA = 4 warps = 64 query rows of one (sequence, head); K/V stream through a
// cp.async double-buffered smem ring in 64-key tiles; online softmax in fp32 (exp2);
// bf16 mma.sync m16n8k16 with fp32 accumulation. head_dim 72 is zero-padded to 80 in smem.
//
// Sequences are addressed through an index map so the same kernel serves every layout
// of the DDiT step without re-layout copies:
//   row(seq i, token j) = (i / inner) * outer + (i % inner) * inner_stride + j * tok
// spatial  (layout [B][t][s]):  inner=1,  outer=S,        tok=1   (frames are sequences)
// temporal (layout [B][t][s]):  inner=Sl, outer=T*Sl, inner_stride=1, tok=Sl
// cross q  (batch b rows):      inner=1,  outer=rows_per_b, tok=1; kv: outer=300, tok=1
#include "common.cuh"
#include "ddit.h"
#include "capi_internal.h"

namespace ddit {

static constexpr int HD = 72;     // head dim
static constexpr int HDP = 80;    // padded to the k16 / n8 granularity
static constexpr int PITCH = 88;  // smem row pitch (elements): 176 B -> conflict-free ldmatrix
static constexpr int BQ = 64;
static constexpr int BKV = 64;
static constexpr int ATT_THREADS = 128;

struct AttnParams {
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  __nv_bfloat16* o;
  int ldq, ldk, ldv, ldo;
  int Lq, Lk;
  int q_inner, q_outer, q_inner_stride, q_tok;
  int kv_inner, kv_outer, kv_inner_stride, kv_tok;
  float scale_log2;  // softmax scale * log2(e)
};

DDIT_DEV void cp_async16(uint32_t smem, const void* g, bool pred) {
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem), "l"(g), "r"(n));
}
DDIT_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
DDIT_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

DDIT_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
DDIT_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
DDIT_DEV void ldsm_x2_t(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(addr));
}
DDIT_DEV void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(addr));
}
DDIT_DEV void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                       uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

DDIT_DEV int seq_row(int i, int inner, int outer, int inner_stride) {
  return (i / inner) * outer + (i % inner) * inner_stride;
}

// Load `rows` tokens (72 bf16 each = 9 x 16 B) of one head into smem [BQ][PITCH].
DDIT_DEV void load_tile(__nv_bfloat16* sm, const __nv_bfloat16* g, int ld, int base_row, int tok,
                        int j0, int L, int col0) {
  const uint32_t s0 = smem_u32(sm);
  for (int c = threadIdx.x; c < 64 * 9; c += ATT_THREADS) {
    const int r = c / 9, ch = c % 9;
    const int j = j0 + r;
    const bool ok = j < L;
    const __nv_bfloat16* src = g + (size_t)(base_row + (ok ? j : 0) * tok) * ld + col0 + ch * 8;
    cp_async16(s0 + (r * PITCH + ch * 8) * 2, src, ok);
  }
}

__global__ void __launch_bounds__(ATT_THREADS)
    flash_attn_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ __align__(16) uint8_t att_smem[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(att_smem);
  __nv_bfloat16* sK[2] = {sQ + BQ * PITCH, sQ + 2 * BQ * PITCH};
  __nv_bfloat16* sV[2] = {sQ + 3 * BQ * PITCH, sQ + 4 * BQ * PITCH};

  const int qb = blockIdx.x, head = blockIdx.y, seq = blockIdx.z;
  const int warp = warp_id(), lane = lane_id();
  const int q0 = qb * BQ;
  const int qbase = seq_row(seq, p.q_inner, p.q_outer, p.q_inner_stride);
  const int kvbase = seq_row(seq, p.kv_inner, p.kv_outer, p.kv_inner_stride);
  const int col0 = head * HD;

  // zero the d-padding columns [72, 80) of Q and K tiles once (never written by cp.async)
  for (int r = threadIdx.x; r < BQ; r += ATT_THREADS) {
    *reinterpret_cast<uint4*>(&sQ[r * PITCH + HD]) = make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint4*>(&sK[0][r * PITCH + HD]) = make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint4*>(&sK[1][r * PITCH + HD]) = make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint4*>(&sV[0][r * PITCH + HD]) = make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint4*>(&sV[1][r * PITCH + HD]) = make_uint4(0, 0, 0, 0);
  }
  load_tile(sQ, p.q, p.ldq, qbase, p.q_tok, q0, p.Lq, col0);
  load_tile(sK[0], p.k, p.ldk, kvbase, p.kv_tok, 0, p.Lk, col0);
  load_tile(sV[0], p.v, p.ldv, kvbase, p.kv_tok, 0, p.Lk, col0);
  cp_async_commit();

  const int nkv = (p.Lk + BKV - 1) / BKV;
  float o[10][4];
#pragma unroll
  for (int i = 0; i < 10; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  uint32_t qa[5][4];

  const int g = lane >> 2, t4 = lane & 3;

  for (int kb = 0; kb < nkv; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nkv) {
      load_tile(sK[buf ^ 1], p.k, p.ldk, kvbase, p.kv_tok, (kb + 1) * BKV, p.Lk, col0);
      load_tile(sV[buf ^ 1], p.v, p.ldv, kvbase, p.kv_tok, (kb + 1) * BKV, p.Lk, col0);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (kb == 0) {
      const uint32_t qaddr = smem_u32(&sQ[(warp * 16 + (lane & 15)) * PITCH + (lane >> 4) * 8]);
#pragma unroll
      for (int ks = 0; ks < 5; ++ks) ldsm_x4(qaddr + ks * 32, qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
    }
    // S = Q K^T for this warp's 16 rows x 64 keys
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
    const __nv_bfloat16* kt = sK[buf];
#pragma unroll
    for (int np = 0; np < 4; ++np) {
      const int key = np * 16 + (lane >> 4) * 8 + (lane & 7);
      const uint32_t kaddr = smem_u32(&kt[key * PITCH + ((lane >> 3) & 1) * 8]);
#pragma unroll
      for (int ks = 0; ks < 5; ++ks) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kaddr + ks * 32, b0, b1, b2, b3);
        mma_bf16(s[2 * np], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
        mma_bf16(s[2 * np + 1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b2, b3);
      }
    }
    // mask keys beyond Lk, online softmax (rows g and g+8 of the warp tile)
    const int kbase = kb * BKV;
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int key = kbase + nt * 8 + 2 * t4;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool ok = key + e < p.Lk;
        s[nt][e] = ok ? s[nt][e] * p.scale_log2 : -INFINITY;
        s[nt][2 + e] = ok ? s[nt][2 + e] * p.scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, s[nt][e]);
        mx1 = fmaxf(mx1, s[nt][2 + e]);
      }
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float c0 = exp2f(m0 - mx0), c1 = exp2f(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      s[nt][0] = exp2f(s[nt][0] - mx0);
      s[nt][1] = exp2f(s[nt][1] - mx0);
      s[nt][2] = exp2f(s[nt][2] - mx1);
      s[nt][3] = exp2f(s[nt][3] - mx1);
      rs0 += s[nt][0] + s[nt][1];
      rs1 += s[nt][2] + s[nt][3];
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      o[i][0] *= c0;
      o[i][1] *= c0;
      o[i][2] *= c1;
      o[i][3] *= c1;
    }
    // O += P V
    const __nv_bfloat16* vt = sV[buf];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t a0 = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      const uint32_t a1 = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      const uint32_t a2 = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      const uint32_t a3 = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
      const int key = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
      for (int dp = 0; dp < 5; ++dp) {
        const uint32_t vaddr = smem_u32(&vt[key * PITCH + dp * 16 + (lane >> 4) * 8]);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vaddr, b0, b1, b2, b3);
        mma_bf16(o[2 * dp], a0, a1, a2, a3, b0, b1);
        mma_bf16(o[2 * dp + 1], a0, a1, a2, a3, b2, b3);
      }
    }
    __syncthreads();
  }
  // finalize
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f;
  const float inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
  const int r0 = q0 + warp * 16 + g;
  const int r1 = r0 + 8;
#pragma unroll
  for (int nt = 0; nt < 9; ++nt) {  // only the 72 real columns
    const int d = nt * 8 + 2 * t4;
    if (r0 < p.Lq) {
      __nv_bfloat16* dst = p.o + (size_t)(qbase + r0 * p.q_tok) * p.ldo + col0 + d;
      *reinterpret_cast<uint32_t*>(dst) = pack_bf16(o[nt][0] * inv0, o[nt][1] * inv0);
    }
    if (r1 < p.Lq) {
      __nv_bfloat16* dst = p.o + (size_t)(qbase + r1 * p.q_tok) * p.ldo + col0 + d;
      *reinterpret_cast<uint32_t*>(dst) = pack_bf16(o[nt][2] * inv1, o[nt][3] * inv1);
    }
  }
}

int attention_launch(const ddit_attn* a, cudaStream_t s) {
  if (a->head_dim != HD) {
    set_error("attention: head_dim %d unsupported (72 only)", a->head_dim);
    return DDIT_E_INVALID;
  }
  if (a->Lq <= 0 || a->Lk <= 0 || a->num_seqs <= 0 || a->heads <= 0 || a->num_seqs > 65535 ||
      a->heads > 65535) {
    set_error("attention: bad sizes Lq=%d Lk=%d seqs=%d heads=%d", a->Lq, a->Lk, a->num_seqs,
              a->heads);
    return DDIT_E_INVALID;
  }
  if ((a->ldq | a->ldk | a->ldv) % 8 != 0) {
    set_error("attention: row strides must be multiples of 8 elements");
    return DDIT_E_INVALID;
  }
  AttnParams p;
  p.q = static_cast<const __nv_bfloat16*>(a->q);
  p.k = static_cast<const __nv_bfloat16*>(a->k);
  p.v = static_cast<const __nv_bfloat16*>(a->v);
  p.o = static_cast<__nv_bfloat16*>(a->o);
  p.ldq = a->ldq;
  p.ldk = a->ldk;
  p.ldv = a->ldv;
  p.ldo = a->ldo;
  p.Lq = a->Lq;
  p.Lk = a->Lk;
  p.q_inner = a->q_inner > 0 ? a->q_inner : 1;
  p.q_outer = a->q_outer;
  p.q_inner_stride = a->q_inner_stride;
  p.q_tok = a->q_tok;
  p.kv_inner = a->kv_inner > 0 ? a->kv_inner : 1;
  p.kv_outer = a->kv_outer;
  p.kv_inner_stride = a->kv_inner_stride;
  p.kv_tok = a->kv_tok;
  p.scale_log2 = a->scale * 1.4426950408889634f;
  dim3 grid((a->Lq + BQ - 1) / BQ, a->heads, a->num_seqs);
  constexpr int smem = 5 * BQ * PITCH * 2;
  static size_t attr[64] = {};
  ensure_smem((const void*)flash_attn_kernel, smem, attr);
  flash_attn_kernel<<<grid, ATT_THREADS, smem, s>>>(p);
  return check_cuda("flash_attn_kernel");
}

}  // namespace ddit

extern "C" DDIT_API int ddit_attention(const ddit_attn* a, void* stream) {
  return ddit::attention_launch(a, static_cast<cudaStream_t>(stream));
}
