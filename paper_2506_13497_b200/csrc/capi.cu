// extern "C" entry points of libddit.so (declared in include/ddit.h).
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "ddit.h"
#include "capi_internal.h"
#include "gemm_sm100.cuh"
#include "elementwise.cuh"

namespace ddit {
static thread_local char g_capi_err[1024] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_capi_err, sizeof g_capi_err, fmt, ap);
  va_end(ap);
}
int check_cuda(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return DDIT_E_CUDA;
  }
  return DDIT_OK;
}
EpiParams to_epi(const ddit_epi* e) {
  EpiParams p;
  memset(&p, 0, sizeof p);
  if (!e) return p;
  p.bias = e->bias;
  p.out = e->out;
  p.ldo = e->ldo;
  p.resid = e->resid;
  p.ldr = e->ldr;
  p.gate = e->gate;
  p.gate_stride = e->gate_stride;
  p.rows_per_b = e->rows_per_b > 0 ? e->rows_per_b : 0x7fffffff;
  p.out2 = static_cast<__nv_bfloat16*>(e->out2);
  p.ldo2 = e->ldo2;
  p.qnorm_w = e->qnorm_w;
  p.knorm_w = e->knorm_w;
  p.hidden = e->hidden;
  p.rope = e->rope;
  p.rope_T = e->rope_T > 0 ? e->rope_T : 1;
  p.rope_S = e->rope_S > 0 ? e->rope_S : 1;
  p.rope_tab = reinterpret_cast<const float2*>(e->rope_tab);
  p.eps = e->eps > 0 ? e->eps : 1e-6f;
  return p;
}
}  // namespace ddit

using namespace ddit;

extern "C" {

DDIT_API const char* ddit_last_error(void) { return g_capi_err; }
DDIT_API int ddit_version(void) { return 1; }
DDIT_API int ddit_num_sms(void) { return num_sms(); }
DDIT_API int ddit_enable_peer_access(int device, int peer) {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(cur);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return DDIT_OK;
  }
  if (e != cudaSuccess) {
    set_error("cudaDeviceEnablePeerAccess(%d -> %d): %s", device, peer, cudaGetErrorString(e));
    return DDIT_E_CUDA;
  }
  return DDIT_OK;
}
DDIT_API int ddit_set_pdl(int on) {
  set_pdl(on);
  return DDIT_OK;
}
DDIT_API int ddit_ln_modulate(const float* x, void* out_bf16, int M, int C, const float* shift,
                              const float* scale, int mod_stride, int rows_per_b, float eps,
                              void* stream) {
  if (!x || !out_bf16 || !shift || !scale) {
    set_error("ddit_ln_modulate: null argument");
    return DDIT_E_INVALID;
  }
  if (ln_modulate(x, static_cast<__nv_bfloat16*>(out_bf16), M, C, shift, scale, mod_stride,
                  rows_per_b, eps, static_cast<cudaStream_t>(stream))) {
    set_error("ddit_ln_modulate: unsupported shape M=%d C=%d", M, C);
    return DDIT_E_INVALID;
  }
  return check_cuda("ln_modulate");
}
DDIT_API int ddit_set_ln_variant(int variant) {
  if (variant < 0 || variant > 5 || variant == 4) {
    set_error("ddit_set_ln_variant: unknown variant %d", variant);
    return DDIT_E_INVALID;
  }
  set_ln_variant(variant);
  return DDIT_OK;
}
DDIT_API int ddit_set_resid_reduce(int on) {
  set_resid_red(on);
  return DDIT_OK;
}
DDIT_API int ddit_set_gemm_2cta(int on) {
  set_two_cta(on);
  return DDIT_OK;
}
DDIT_API int ddit_set_gemm_wide(int on) {
  set_gemm_wide(on);
  return DDIT_OK;
}

DDIT_API int ddit_gemm(const void* A, int lda, const void* B, int ldb, int M, int N, int K, int epi,
                       const ddit_epi* ep, int bn, void* stream) {
  GemmPlan plan;
  int rc = gemm_plan_init(&plan, A, lda, B, ldb, M, N, K, epi, to_epi(ep), bn);
  if (rc) {
    set_error("ddit_gemm: %s", gemm_last_error());
    return rc == -3 ? DDIT_E_TMA : DDIT_E_INVALID;
  }
  rc = gemm_plan_launch(&plan, static_cast<cudaStream_t>(stream));
  if (rc) {
    set_error("ddit_gemm: %s", gemm_last_error());
    return DDIT_E_CUDA;
  }
  return DDIT_OK;
}

}  // extern "C"
