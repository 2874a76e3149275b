// LN+modulate at the 240p shape: current warp-per-row two-pass kernel vs a streaming kernel that
// gets (mean, rstd) per row precomputed (what a stats-producing residual epilogue would allow)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) { __nv_bfloat162 v = __floats2bfloat162_rn(a, b); return *reinterpret_cast<uint32_t*>(&v); }
__device__ __forceinline__ float warp_sum(float v) { for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o); return v; }
__global__ void __launch_bounds__(128) ln_cur(const float* __restrict__ x, __nv_bfloat16* __restrict__ out, int M, int C,
    const float* __restrict__ shift, const float* __restrict__ scale, int rows_per_b, float eps) {
  const int row = blockIdx.x * 4 + (threadIdx.x / 32), lane = threadIdx.x & 31;
  if (row >= M) return;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)row * C);
  float4 v[9]; float s = 0.f;
#pragma unroll
  for (int i = 0; i < 9; ++i) { v[i] = __ldcs(xr + lane + 32 * i); s += (v[i].x + v[i].y) + (v[i].z + v[i].w); }
  const float mean = warp_sum(s) / C; float q = 0.f;
#pragma unroll
  for (int i = 0; i < 9; ++i) { float a = v[i].x - mean, b = v[i].y - mean, c = v[i].z - mean, d = v[i].w - mean; q += (a*a + b*b) + (c*c + d*d); }
  const float rstd = rsqrtf(warp_sum(q) / C + eps);
  const int bi = row / rows_per_b;
  const float4* sh = reinterpret_cast<const float4*>(shift + (size_t)bi * 6 * C);
  const float4* sc = reinterpret_cast<const float4*>(scale + (size_t)bi * 6 * C);
  uint2* o = reinterpret_cast<uint2*>(out + (size_t)row * C);
#pragma unroll
  for (int i = 0; i < 9; ++i) { const int c = lane + 32 * i; const float4 a = __ldg(sh + c), k = __ldg(sc + c);
    o[c] = make_uint2(pack_bf16((v[i].x - mean) * rstd * (1.f + k.x) + a.x, (v[i].y - mean) * rstd * (1.f + k.y) + a.y),
                      pack_bf16((v[i].z - mean) * rstd * (1.f + k.z) + a.z, (v[i].w - mean) * rstd * (1.f + k.w) + a.w)); }
}
// streaming: each thread 4 float4 of one row segment; stats (mean, rstd) given
__global__ void __launch_bounds__(256) ln_stream(const float* __restrict__ x, __nv_bfloat16* __restrict__ out, int M, int C,
    const float* __restrict__ shift, const float* __restrict__ scale, int rows_per_b, const float2* __restrict__ st) {
  const int nv = C / 4;
  const long long total = (long long)M * nv;
  for (long long i0 = (long long)blockIdx.x * blockDim.x * 4 + threadIdx.x; i0 < total; i0 += (long long)gridDim.x * blockDim.x * 4) {
    float4 v[4]; int rr[4], cc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) { long long i = i0 + k * blockDim.x; rr[k] = i < total ? (int)(i / nv) : 0; cc[k] = (int)(i - (long long)rr[k] * nv);
      if (i < total) v[k] = __ldcs(reinterpret_cast<const float4*>(x) + i); }
#pragma unroll
    for (int k = 0; k < 4; ++k) { long long i = i0 + k * blockDim.x; if (i >= total) break;
      const float2 ms = __ldg(st + rr[k]); const int bi = rr[k] / rows_per_b;
      const float4 a = __ldg(reinterpret_cast<const float4*>(shift + (size_t)bi * 6 * C) + cc[k]);
      const float4 g = __ldg(reinterpret_cast<const float4*>(scale + (size_t)bi * 6 * C) + cc[k]);
      reinterpret_cast<uint2*>(out)[i] = make_uint2(pack_bf16((v[k].x - ms.x) * ms.y * (1.f + g.x) + a.x, (v[k].y - ms.x) * ms.y * (1.f + g.y) + a.y),
                                                    pack_bf16((v[k].z - ms.x) * ms.y * (1.f + g.z) + a.z, (v[k].w - ms.x) * ms.y * (1.f + g.w) + a.w)); }
  }
}
int main() {
  const int M = 12150, C = 1152;
  float *x, *mod; __nv_bfloat16* out; float2* st;
  cudaMalloc(&x, (size_t)M * C * 4); cudaMalloc(&out, (size_t)M * C * 2); cudaMalloc(&mod, 2 * 6 * C * 4); cudaMalloc(&st, M * 8);
  cudaMemset(x, 0, (size_t)M * C * 4); cudaMemset(mod, 0, 2 * 6 * C * 4); cudaMemset(st, 0, M * 8);
  float* flush; cudaMalloc(&flush, 256 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int variant = 0; variant < 3; ++variant) {
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      cudaMemset(flush, r, 256 << 20);  // evict x from L2 (cold, like ncu)
      cudaEventRecord(a);
      if (variant == 0) ln_cur<<<(M + 3) / 4, 128>>>(x, out, M, C, mod, mod + C, M / 2, 1e-6f);
      else if (variant == 1) ln_stream<<<148 * 8, 256>>>(x, out, M, C, mod, mod + C, M / 2, st);
      else ln_stream<<<148 * 16, 256>>>(x, out, M, C, mod, mod + C, M / 2, st);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("%s: %.1f us  %.2f TB/s\n", variant == 0 ? "current two-pass" : variant == 1 ? "streaming g1184" : "streaming g2368", best * 1e3, (double)M * C * 6 / (best * 1e-3) / 1e12);
  }
  // warm (x in L2): no flush
  for (int variant = 0; variant < 2; ++variant) {
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(a);
      if (variant == 0) ln_cur<<<(M + 3) / 4, 128>>>(x, out, M, C, mod, mod + C, M / 2, 1e-6f);
      else ln_stream<<<148 * 8, 256>>>(x, out, M, C, mod, mod + C, M / 2, st);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("warm %s: %.1f us\n", variant == 0 ? "current" : "streaming", best * 1e3);
  }
}
