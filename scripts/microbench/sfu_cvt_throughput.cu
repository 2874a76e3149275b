// throughput of ex2.approx.f32, ex2.approx.f16x2, cvt.rn.bf16x2.f32 (F2FP), FFMA2 per SM
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
template <int OP>
__global__ void k(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  uint32_t u[8] = {0};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) { asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[i])); }
      if (OP == 2) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i+1)&7])); u[i] ^= r; a[i] += 1e-7f; }
      if (OP == 3) { asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i])); }
      if (OP == 4) { uint32_t r; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i+1)&7])); u[i] ^= r; a[i] += 1e-7f; }
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + (float)u[i];
  if (s == 1234.5f) out[0] = s;
}
int main() {
  float* d; cudaMalloc(&d, 4);
  const char* names[] = {"ex2.f32", "ex2.f16x2", "cvt.bf16x2.f32", "ffma", "cvt.f16x2.f32"};
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int op = 0; op < 5; ++op) {
    int iters = 4096;
    auto f = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : k<4>;
    f<<<sms * 4, 256>>>(d, iters);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    f<<<sms * 4, 256>>>(d, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)sms * 4 * 256 * iters * 8;
    printf("%-16s %.2f Gop/s total, %.1f ops/clk/SM at %d MHz nominal\n", names[op], ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
}
