// Latent re-sharding between DoP groups:
//   * promotion P -> P' at a step boundary (reference engine.py:281-290, where the simulator
//     charges a constant 1 ms broadcast + 1 ms scale-up): every rank of the new group pulls the
//     frames of its new T-shard from whichever old ranks hold them;
//   * DiT -> VAE hand-off (reference policies.py:175-190 / allocator.py:279-321): the
//     vae_dop lowest-id GPUs gather the whole latent (or their frame range) from the DiT group.
// z shards are channel-major [Cin][Tl][Hl][Wl] fp32, so one (channel, frame) is a contiguous
// Hl*Wl run; sources are peer pointers (NVLink) or local buffers. One warp per (channel,
// frame) run, 16-byte vectors when aligned.
#include "common.cuh"
#include "ddit.h"
#include "capi_internal.h"

#include <cstring>

namespace ddit {

struct GatherSrc {
  const float* p[16];
  int t_lo[16], t_hi[16];
  int n;
};

__global__ void __launch_bounds__(256)
    latent_gather_kernel(float* __restrict__ dst, int t_lo, int t_hi, GatherSrc src, int Cin,
                         int HW) {
  const int Tl = t_hi - t_lo;
  const int runs = Cin * Tl;
  for (int run = blockIdx.x * 8 + (threadIdx.x >> 5); run < runs; run += gridDim.x * 8) {
    const int c = run / Tl, t = t_lo + run % Tl;
    int k = 0;
    while (k < src.n && !(t >= src.t_lo[k] && t < src.t_hi[k])) ++k;
    if (k == src.n) continue;  // unreachable when the sources cover [t_lo, t_hi)
    const int sTl = src.t_hi[k] - src.t_lo[k];
    const float* s = src.p[k] + ((size_t)c * sTl + (t - src.t_lo[k])) * HW;
    float* d = dst + ((size_t)c * Tl + (t - t_lo)) * HW;
    const int lane = threadIdx.x & 31;
    if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0) {
      const int n4 = HW >> 2;
      for (int i = lane; i < n4; i += 32)
        reinterpret_cast<float4*>(d)[i] = reinterpret_cast<const float4*>(s)[i];
      for (int i = (n4 << 2) + lane; i < HW; i += 32) d[i] = s[i];
    } else {
      for (int i = lane; i < HW; i += 32) d[i] = s[i];
    }
  }
}

}  // namespace ddit

extern "C" DDIT_API int ddit_latent_gather(float* dst, int t_lo, int t_hi, const float* const* src,
                                           const int* src_t_lo, const int* src_t_hi, int nsrc,
                                           int channels, int hw, void* stream) {
  using namespace ddit;
  if (nsrc < 1 || nsrc > 16 || t_hi < t_lo || channels < 1 || hw < 1) {
    set_error("latent_gather: bad arguments (nsrc %d in [1,16])", nsrc);
    return DDIT_E_INVALID;
  }
  GatherSrc g;
  memset(&g, 0, sizeof g);
  g.n = nsrc;
  for (int k = 0; k < nsrc; ++k) {
    g.p[k] = src[k];
    g.t_lo[k] = src_t_lo[k];
    g.t_hi[k] = src_t_hi[k];
  }
  // coverage check on the host: every destination frame must have a source
  for (int t = t_lo; t < t_hi; ++t) {
    bool ok = false;
    for (int k = 0; k < nsrc && !ok; ++k) ok = t >= g.t_lo[k] && t < g.t_hi[k];
    if (!ok) {
      set_error("latent_gather: frame %d has no source shard", t);
      return DDIT_E_INVALID;
    }
  }
  const int runs = channels * (t_hi - t_lo);
  if (runs == 0) return DDIT_OK;
  int grid = (runs + 7) / 8;
  if (grid > 1184) grid = 1184;
  latent_gather_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(dst, t_lo, t_hi, g,
                                                                             channels, hw);
  return check_cuda("latent_gather_kernel");
}
