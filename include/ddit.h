/*
 * ddit.h -- C ABI of the B200-native DDiT hot path (libddit.so, sm_100a).
 *
 * The reference (arxiv 2506.13497, `ditsim`) has no FFI: the hot path is the Python
 * duck-typed execution model `ProfileTable.dit_step(resolution, dop) -> seconds`
 * (reference pkg/src/ditsim/profiles.py:69-76, called from engine.py:245,289,292) and
 * `ProfileTable.vae(resolution, dop)` (profiles.py:78-85, engine.py:305). This header is the
 * native boundary that replaces those lookups with real work on B200s: every entry point takes
 * plain device pointers, sizes and a cudaStream_t (passed as void*), returns 0 on success or a
 * negative DDIT_E* code, and never throws. `ddit_last_error()` gives the message of the last
 * failure on the calling thread. Only the controller thread of a process calls in.
 *
 * Python binds it with ctypes (paper_2506_13497_b200/_lib.py); INTEGRATION.md shows the
 * binding a ditsim maintainer would add.
 */
#ifndef DDIT_H_
#define DDIT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DDIT_API __attribute__((visibility("default")))

/* Error codes. Python maps DDIT_E_LOOKUP -> ProfileLookupError (profiles.py:36-37),
 * DDIT_E_ALLOC -> AllocationError (allocator.py:22-23), DDIT_E_CONFIG -> SimulationError
 * (engine.py:33-34); the others raise RuntimeError. */
#define DDIT_OK 0
#define DDIT_E_INVALID (-2)  /* bad argument / shape */
#define DDIT_E_TMA (-3)      /* tensor-map creation failed */
#define DDIT_E_CUDA (-4)     /* CUDA runtime error */
#define DDIT_E_LOOKUP (-5)   /* unknown resolution / DoP */
#define DDIT_E_ALLOC (-6)    /* device memory / group misuse */
#define DDIT_E_CONFIG (-7)   /* inconsistent configuration */

DDIT_API const char* ddit_last_error(void);
DDIT_API int ddit_version(void);
DDIT_API int ddit_num_sms(void);

/* ------------------------------------------------------------------ kernel-level ops
 * Exposed for parity tests and profiling; the step below composes them. */

/* Epilogue kinds of ddit_gemm (see csrc/gemm_sm100.cuh). */
#define DDIT_EPI_BF16 0      /* out_bf16 = A.B^T + bias */
#define DDIT_EPI_GELU_BF16 1 /* out_bf16 = gelu_tanh(A.B^T + bias) */
#define DDIT_EPI_RESID 2     /* resid_f32 += gate[b] * (A.B^T + bias) (+ bf16 copy) */
#define DDIT_EPI_QKV 3       /* bias + per-head RMSNorm on q,k + optional RoPE; bf16 out */
#define DDIT_EPI_F32 4       /* out_f32 = A.B^T + bias */

typedef struct ddit_epi {
  const float* bias;   /* [N] fp32 or NULL */
  void* out;           /* bf16 [M, ldo] (DDIT_EPI_F32: fp32) */
  int ldo;
  float* resid;        /* DDIT_EPI_RESID: fp32 [M, ldr] */
  int ldr;
  const float* gate;   /* DDIT_EPI_RESID: fp32 [B][gate_stride] or NULL (gate = 1) */
  int gate_stride;
  int rows_per_b;      /* row r belongs to batch r / rows_per_b */
  void* out2;          /* DDIT_EPI_RESID: optional bf16 copy of the new residual */
  int ldo2;
  const float* qnorm_w; /* DDIT_EPI_QKV: [72] */
  const float* knorm_w; /* DDIT_EPI_QKV: [72] */
  int hidden;          /* DDIT_EPI_QKV: C (q = cols [0,C), k = [C,2C), v = [2C,3C)) */
  int rope;            /* DDIT_EPI_QKV: 1 = rotate q,k by frame index */
  int rope_T;          /* frames */
  int rope_S;          /* rows per frame in this layout: t = (row / rope_S) % rope_T */
  const float* rope_tab; /* [rope_T][36][2] (cos, sin) */
  float eps;
} ddit_epi;

/* D = A[M,K] . B[N,K]^T on tcgen05 (bf16 in, fp32 accumulate) with a fused epilogue.
 * bn in {128,144,192,256}; N % bn == 0; K % 64 == 0. */
DDIT_API int ddit_gemm(const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                       int epi, const ddit_epi* ep, int bn, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DDIT_H_ */
