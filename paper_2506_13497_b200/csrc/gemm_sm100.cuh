// Host-visible declarations for the tcgen05 GEMM (D = A . B^T, bf16 in, fp32 acc) with the
// fused STDiT epilogues. Layout contract: A [M, K] row-major (K contiguous, row stride lda),
// B [N, K] row-major (nn.Linear weight layout), both staged K-major by TMA with the 128 B swizzle.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace ddit {

enum EpiKind : int {
  EPI_BF16 = 0,       // out_bf16 = acc + bias
  EPI_GELU_BF16 = 1,  // out_bf16 = gelu_tanh(acc + bias)
  EPI_RESID = 2,      // resid_f32 += gate[b] * (acc + bias)   (gate == null -> 1); optional bf16 copy
  EPI_QKV = 3,        // out_bf16 = rope(rmsnorm_head(acc + bias)) on the q/k sections; v: acc + bias
  EPI_F32 = 4,        // out_f32 = acc + bias
  EPI_RESID_COPY = 5, // internal: EPI_RESID with the bf16 copy, stored in 64-column (128 B) boxes
  EPI_RESID_RED = 6,  // internal: EPI_RESID without copy / exchange: gate * (acc + bias) leaves
                      // through a TMA reduce-add into resid (the L2 does x + y; nothing is loaded)
};

struct EpiParams {
  const float* bias;        // [N] or null
  void* out;                // bf16 [M, ldo] (EPI_F32: fp32)
  int ldo;
  float* resid;             // EPI_RESID: fp32 [M, ldr]
  int ldr;
  const float* gate;        // EPI_RESID: [B][gate_stride] or null
  int gate_stride;
  int rows_per_b;           // row -> batch index b = row / rows_per_b
  __nv_bfloat16* out2;      // EPI_RESID: optional bf16 copy of the updated residual [M, ldo2]
  int ldo2;
  // EPI_QKV
  const float* qnorm_w;     // [head_dim]
  const float* knorm_w;     // [head_dim]
  int hidden;               // C: q = [0,C), k = [C,2C), v = [2C,3C)
  int rope;                 // 1: rotate q,k by frame position
  int rope_T;               // number of frames
  int rope_S;               // tokens per frame in this row layout: t = (row / rope_S) % rope_T
  const float2* rope_tab;   // [rope_T][head_dim/2] (cos, sin)
  float eps;
  // EPI_RESID with the DSP exchange fused in (xch != 0): the updated rows are stored straight
  // into their owner rank's buffer of the other layout (peer memory) instead of back into
  // resid, and the last CTA publishes the exchange flag (layouts: exchange.cu)
  int xch;                  // 0: none, 1: x_sp -> x_tp (spatial block), 2: x_tp -> x_sp (temporal)
  float* xdst[8];           // destination buffer of every rank
  int xB, xT, xS, xP;       // CFG batch, frames, tokens per frame, DoP
  int xlo, xlen, xchunk;    // 1: t_lo, Tl, ceil(S/P); 2: s_lo, Sl, ceil(T/P)
  uint32_t* xflags[8];      // every rank's flag array; all null: ranks ordered by the stream
  unsigned int* xcounter;   // CTA ticket counter (zero between exchanges)
  uint32_t* xepoch;         // this rank's exchange epoch
  int xrank;
};

struct GemmPlan {
  CUtensorMap tmA;
  CUtensorMap tmB;
  CUtensorMap tmO;   // epilogue output (bf16 / f32 / qkv)
  CUtensorMap tmR;   // fp32 residual (EPI_RESID)
  CUtensorMap tmO2;  // bf16 copy of the residual (EPI_RESID, optional)
  int M, N, K;
  int bn;
  int epi;
  EpiParams ep;
  int grid;
  int two_cta;  // 1: cta_group::2 kernel (M = 256 tiles over a CTA pair)
  int wide;     // 1: 2-CTA tiles of 256 x 2BN (two accumulator halves, one tile in TMEM)
};

// Build the TMA descriptors and launch geometry. Returns 0 on success.
int gemm_plan_init(GemmPlan* p, const void* A, int lda, const void* B, int ldb, int M, int N,
                   int K, int epi, const EpiParams& ep, int bn);
int gemm_plan_init_cta(GemmPlan* p, const void* A, int lda, const void* B, int ldb, int M, int N,
                       int K, int epi, const EpiParams& ep, int bn, int two_cta);
// BN and 1-/2-CTA tiles for an M x N output (fills the GPU at small M; bit-identical results)
void gemm_pick_tile(int M, int N, int epi, int* bn, int* two_cta);
int gemm_plan_launch(const GemmPlan* p, cudaStream_t stream);
// recompute the tile shape / grid after editing p->ep (e.g. attaching the DSP exchange)
void gemm_plan_refresh(GemmPlan* p);
int num_sms();
bool two_cta_enabled();
bool gemm_wide_enabled();
void set_gemm_wide(int on);
bool resid_red_enabled();
void set_resid_red(int on);
void set_pdl(int on);
void set_two_cta(int on);
const char* gemm_last_error();

}  // namespace ddit
