// isolated cost of the FMHA softmax exps phase (128 scores -> packed bf16 P) per warp
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#define DDIT_DEV __device__ __forceinline__
DDIT_DEV void ffma2(float& d0, float& d1, float a0, float a1, float b, float c) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\tmov.b64 rc, {%5, %5};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b), "f"(c));
}
DDIT_DEV float2 exp2_poly_x2(float x0, float x1) {
  const float2 x = make_float2(fmaxf(x0, -127.f), fmaxf(x1, -127.f));
  const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 q = __ffma2_rn(make_float2(0.05502926645f, 0.05502926645f), f, make_float2(0.24225698193f, 0.24225698193f));
  q = __ffma2_rn(q, f, make_float2(0.69325305500f, 0.69325305500f));
  q = __ffma2_rn(q, f, make_float2(0.99995133866f, 0.99995133866f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}
DDIT_DEV float fast_exp2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
DDIT_DEV uint32_t pack_bf16(float a, float b) { __nv_bfloat162 v = __floats2bfloat162_rn(a, b); return *reinterpret_cast<uint32_t*>(&v); }
template <int POLY> __host__ __device__ constexpr bool poly_chunk(int c) { return POLY > 0 && c % POLY == POLY - 1; }

template <int POLY>
__global__ void __launch_bounds__(128) k(const float* in, uint32_t* out, long long* cyc, int iters, float scale) {
  uint32_t s[128];
  for (int i = 0; i < 128; ++i) s[i] = __float_as_uint(in[(threadIdx.x * 131 + i) & 1023]);
  float neg_m = -3.f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t sv[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) sv[i] = s[i];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      float pv[8];
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        float x0, x1;
        ffma2(x0, x1, __uint_as_float(sv[c * 8 + e]), __uint_as_float(sv[c * 8 + e + 1]), scale, neg_m);
        if (poly_chunk<POLY>(c)) { const float2 y = exp2_poly_x2(x0, x1); pv[e] = y.x; pv[e + 1] = y.y; }
        else { pv[e] = fast_exp2(x0); pv[e + 1] = fast_exp2(x1); }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) sv[4 * c + e] = pack_bf16(pv[2 * e], pv[2 * e + 1]);
    }
#pragma unroll
    for (int i = 0; i < 64; ++i) acc ^= sv[i];
    neg_m -= 1e-6f;
  }
  long long t1 = clock64();
  out[blockIdx.x * 128 + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int POLY>
__global__ void __launch_bounds__(128) kb(const float* in, uint32_t* out, long long* cyc, int iters, float scale) {
  uint32_t s[128];
  for (int i = 0; i < 128; ++i) s[i] = __float_as_uint(in[(threadIdx.x * 131 + i) & 1023]);
  float neg_m = -3.f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float v[128];
#pragma unroll
    for (int i = 0; i < 128; i += 2) ffma2(v[i], v[i + 1], __uint_as_float(s[i]), __uint_as_float(s[i + 1]), scale, neg_m);
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      if (poly_chunk<POLY>(c)) {
#pragma unroll
        for (int e = 0; e < 8; e += 2) { const float2 y = exp2_poly_x2(v[c * 8 + e], v[c * 8 + e + 1]); v[c * 8 + e] = y.x; v[c * 8 + e + 1] = y.y; }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[c * 8 + e] = fast_exp2(v[c * 8 + e]);
      }
    }
    uint32_t pk[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) pk[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
#pragma unroll
    for (int i = 0; i < 64; ++i) acc ^= pk[i];
    neg_m -= 1e-6f;
  }
  long long t1 = clock64();
  out[blockIdx.x * 128 + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int POLY>
__global__ void __launch_bounds__(128) kc(const float* in, uint32_t* out, long long* cyc, int iters, float scale) {
  uint32_t s[128];
  for (int i = 0; i < 128; ++i) s[i] = __float_as_uint(in[(threadIdx.x * 131 + i) & 1023]);
  float neg_m = -3.f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t sv[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) sv[i] = s[i];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      float pv[8];
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        const float x0 = fmaf(__uint_as_float(sv[c * 8 + e]), scale, neg_m);
        const float x1 = fmaf(__uint_as_float(sv[c * 8 + e + 1]), scale, neg_m);
        if (poly_chunk<POLY>(c)) { const float2 y = exp2_poly_x2(x0, x1); pv[e] = y.x; pv[e + 1] = y.y; }
        else { pv[e] = fast_exp2(x0); pv[e + 1] = fast_exp2(x1); }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) sv[4 * c + e] = pack_bf16(pv[2 * e], pv[2 * e + 1]);
    }
#pragma unroll
    for (int i = 0; i < 64; ++i) acc ^= sv[i];
    neg_m -= 1e-6f;
  }
  long long t1 = clock64();
  out[blockIdx.x * 128 + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* in; uint32_t* out; long long* cyc;
  cudaMalloc(&in, 4096); cudaMalloc(&out, 148 * 128 * 4 * 4); cudaMalloc(&cyc, 148 * 8);
  cudaMemset(in, 0, 4096);
  long long h[148];
  auto run = [&](void (*f)(const float*, uint32_t*, long long*, int, float), const char* name) {
    f<<<148, 128>>>(in, out, cyc, 200, 0.12f);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 148 * 8, cudaMemcpyDeviceToHost);
    printf("%s: %.0f cycles\n", name, (double)h[0] / 200);
  };
  run(kc<0>, "scalar POLY=0"); run(kc<3>, "scalar POLY=3"); run(kc<4>, "scalar POLY=4");
  run(kc<5>, "scalar POLY=5"); run(kc<6>, "scalar POLY=6"); run(kc<8>, "scalar POLY=8");
  run(k<4>, "ffma2 POLY=4"); run(k<6>, "ffma2 POLY=6"); run(k<8>, "ffma2 POLY=8");
}
