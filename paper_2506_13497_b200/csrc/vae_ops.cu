// Memory-bound and small-channel kernels of the VAE decoder, all on
// channels-last activations [N][P][C] (N samples, P = T*H*W pixels):
//   GroupNorm statistics (deterministic: per-block fp32 partials, fixed-order fp64 sum) + normalise / affine /
//   optional SiLU; nearest 2x spatial upsample; depth-to-time (OpenSora temporal upsampler
//   "B (C ts) T H W -> B C (T ts) H W"); direct convolutions for the few layers with fewer than
//   64 channels on one side (latent in, frames out); row softmax and transpose for the
//   decoder's single-head mid-block attention; elementwise add.
#include "common.cuh"
#include "ddit.h"
#include "capi_internal.h"

namespace ddit {

// ------------------------------------------------------------------ GroupNorm
// Deterministic two-level statistics (fixed reduction order: bitwise reproducible).
// gn_partial: block (blk, n) reduces pixels [blk*ppb, (blk+1)*ppb) of sample n into
// partial[n][blk][g] = (sum, sumsq); thread t owns the 8-channel vector t % (C/8) (C/8 divides
// 256) and walks pixels with stride 256 / (C/8).
__global__ void __launch_bounds__(256)
    gn_partial_kernel(const __nv_bfloat16* __restrict__ x, float2* __restrict__ partial, int P,
                      int C, int G, int ppb, int nblk) {
  const int n = blockIdx.y, blk = blockIdx.x;
  const int cg = C / G;
  const int vecs = C / 8;
  const int step = 256 / vecs;
  const int v = threadIdx.x % vecs;
  const int p0 = blk * ppb;
  const int p1 = min(p0 + ppb, P);
  __shared__ float red_s[256][9], red_q[256][9];
  float sg[8], qg[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) sg[e] = qg[e] = 0.f;
  for (int p = p0 + (int)threadIdx.x / vecs; p < p1; p += step) {
    const uint4 u = *reinterpret_cast<const uint4*>(x + ((size_t)n * P + p) * C + v * 8);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = unpack_bf16(w[e]);
      sg[2 * e] += f.x;
      sg[2 * e + 1] += f.y;
      qg[2 * e] += f.x * f.x;
      qg[2 * e + 1] += f.y * f.y;
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    red_s[threadIdx.x][e] = sg[e];
    red_q[threadIdx.x][e] = qg[e];
  }
  __syncthreads();
  if (threadIdx.x < G) {
    const int g = threadIdx.x;
    float s = 0.f, q = 0.f;
    for (int t = 0; t < 256; ++t) {
      const int c0 = (t % vecs) * 8;
      if (c0 + 8 <= g * cg || c0 >= (g + 1) * cg) continue;
      for (int e = 0; e < 8; ++e)
        if ((c0 + e) / cg == g) {
          s += red_s[t][e];
          q += red_q[t][e];
        }
    }
    partial[((size_t)n * nblk + blk) * G + g] = make_float2(s, q);
  }
}

__global__ void gn_finalize_kernel(const float2* __restrict__ partial, double* __restrict__ stats,
                                   int G, int nblk) {
  const int n = blockIdx.x, g = threadIdx.x;
  if (g >= G) return;
  double s = 0, q = 0;
  for (int b = 0; b < nblk; ++b) {
    const float2 v = partial[((size_t)n * nblk + b) * G + g];
    s += v.x;
    q += v.y;
  }
  stats[(n * G + g) * 2] = s;
  stats[(n * G + g) * 2 + 1] = q;
}

// y = act((x - mean) * rstd * gamma + beta), act = SiLU or identity; bf16 in / out.
__global__ void __launch_bounds__(256)
    gn_apply_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                    const double* __restrict__ stats, const float* __restrict__ gamma,
                    const float* __restrict__ beta, int P, int C, int G, float eps, int silu_act,
                    size_t total_vecs) {
  const int cg = C / G;
  const int vecs = C / 8;
  const double cnt = (double)P * cg;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total_vecs;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t pix = i / vecs;
    const int c0 = (int)(i % vecs) * 8;
    const int n = (int)(pix / P);
    const uint4 u = reinterpret_cast<const uint4*>(x)[i];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = unpack_bf16(w[e]);
      float r[2] = {f.x, f.y};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = c0 + 2 * e + h;
        const int g = c / cg;
        const double s = stats[(n * G + g) * 2], q = stats[(n * G + g) * 2 + 1];
        const double mean = s / cnt;
        const double var = fmax(q / cnt - mean * mean, 0.0);
        const float rstd = rsqrtf((float)var + eps);
        float v = (r[h] - (float)mean) * rstd * gamma[c] + beta[c];
        if (silu_act) v = v / (1.f + __expf(-v));
        r[h] = v;
      }
      o[e] = pack_bf16(r[0], r[1]);
    }
    reinterpret_cast<uint4*>(y)[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// ------------------------------------------------------------------ layout ops
// nearest 2x upsample in H and W: [N][H][W][C] -> [N][2H][2W][C]
__global__ void upsample2x_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                  int N, int H, int W, int C) {
  const int vecs = C / 8;
  const size_t total = (size_t)N * 2 * H * 2 * W * vecs;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int v = (int)(i % vecs);
    size_t r = i / vecs;
    const int ox = (int)(r % (2 * W));
    r /= 2 * W;
    const int oy = (int)(r % (2 * H));
    const size_t n = r / (2 * H);
    reinterpret_cast<uint4*>(y)[i] =
        reinterpret_cast<const uint4*>(x)[((n * H + oy / 2) * W + ox / 2) * vecs + v];
  }
}

// [B][T][HW][2C] (channel k = 2c + ts) -> [B][2T][HW][C]
__global__ void depth_to_time_kernel(const __nv_bfloat16* __restrict__ x,
                                     __nv_bfloat16* __restrict__ y, int B, int T, int HW, int C) {
  const size_t total = (size_t)B * 2 * T * HW * C;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    size_t r = i / C;
    const int p = (int)(r % HW);
    r /= HW;
    const int t2 = (int)(r % (2 * T));
    const size_t b = r / (2 * T);
    const int t = t2 >> 1, ts = t2 & 1;
    y[i] = x[(((b * T + t) * HW + p) * (size_t)(2 * C)) + 2 * c + ts];
  }
}

// ------------------------------------------------------------------ small-channel conv
// Direct conv for layers with < 64 channels on one side. x: any strided 5-D layout
// (element strides xs = {b, c, t, h, w}; bf16 or fp32), w: fp32 [Cout][kt][kh][kw][Cin],
// y: [B][T][H][W][Cout] bf16, or fp32 channels-first [B][Cout][T][Hc][Wc] cropped to (Hc, Wc)
// when out_cf is set (the decoded frames).
struct XStrides {
  long long b, c, t, h, w;
};
template <typename TIn>
__global__ void __launch_bounds__(128)
    conv_small_kernel(const TIn* __restrict__ x, XStrides xs, const float* __restrict__ w,
                      const float* __restrict__ bias, void* __restrict__ y, int B, int T, int H,
                      int W, int Cin, int Cout, int kt, int kh, int kw, int pt, int out_cf, int Hc,
                      int Wc) {
  const size_t pix = blockIdx.x * (size_t)blockDim.y + threadIdx.y;
  const size_t npix = (size_t)B * T * H * W;
  if (pix >= npix) return;
  const int xq = (int)(pix % W);
  size_t r = pix / W;
  const int yq = (int)(r % H);
  r /= H;
  const int tq = (int)(r % T);
  const int b = (int)(r / T);
  for (int co = threadIdx.x; co < Cout; co += blockDim.x) {
    float acc = bias ? bias[co] : 0.f;
    for (int dt = 0; dt < kt; ++dt) {
      const int ti = tq + dt - pt;
      if (ti < 0 || ti >= T) continue;
      for (int dy = 0; dy < kh; ++dy) {
        const int yi = yq + dy - kh / 2;
        if (yi < 0 || yi >= H) continue;
        for (int dx = 0; dx < kw; ++dx) {
          const int xi = xq + dx - kw / 2;
          if (xi < 0 || xi >= W) continue;
          const TIn* xp = x + b * xs.b + ti * xs.t + yi * xs.h + xi * xs.w;
          const float* wp = w + ((((size_t)co * kt + dt) * kh + dy) * kw + dx) * Cin;
          for (int ci = 0; ci < Cin; ++ci) acc += wp[ci] * static_cast<float>(xp[ci * xs.c]);
        }
      }
    }
    if (out_cf) {
      if (yq < Hc && xq < Wc)
        static_cast<float*>(y)[((((size_t)b * Cout + co) * T + tq) * Hc + yq) * Wc + xq] = acc;
    } else {
      static_cast<__nv_bfloat16*>(y)[pix * Cout + co] = __float2bfloat16(acc);
    }
  }
}

// ------------------------------------------------------------------ mid-block attention helpers
// P[r, c] = softmax_c(S[r, c] * scale) over c < valid, 0 for padded columns. S fp32, P bf16.
__global__ void __launch_bounds__(256)
    softmax_rows_kernel(const float* __restrict__ S, __nv_bfloat16* __restrict__ P, int rows,
                        int cols, int valid, float scale) {
  const int r = blockIdx.x;
  if (r >= rows) return;
  const float* s = S + (size_t)r * cols;
  __shared__ float red[32];
  float m = -INFINITY;
  for (int c = threadIdx.x; c < valid; c += blockDim.x) m = fmaxf(m, s[c] * scale);
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : -INFINITY;
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  m = red[0];
  __syncthreads();
  float sum = 0.f;
  for (int c = threadIdx.x; c < valid; c += blockDim.x) sum += __expf(s[c] * scale - m);
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = 1.f / red[0];
  for (int c = threadIdx.x; c < cols; c += blockDim.x)
    P[(size_t)r * cols + c] = __float2bfloat16(c < valid ? __expf(s[c] * scale - m) * inv : 0.f);
}

// out[c][r] = in[r][c] (rows x cols, ld_in) into ld_out; bf16; zero-fills columns r >= rows
// up to rows_pad.
__global__ void transpose_kernel(const __nv_bfloat16* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                 int rows, int cols, int ld_in, int rows_pad) {
  __shared__ __nv_bfloat16 tile[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? in[(size_t)r * ld_in + c] : __float2bfloat16(0.f);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols && r < rows_pad) out[(size_t)c * rows_pad + r] = tile[threadIdx.x][i];
  }
}

// y = bf16(a_f32 + b_bf16)
__global__ void add_f32_bf16_kernel(const float* __restrict__ a, const __nv_bfloat16* __restrict__ b,
                                    __nv_bfloat16* __restrict__ y, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16(a[i] + __bfloat162float(b[i]));
}

static int blocks_for(size_t n, int tpb) {
  size_t b = (n + tpb - 1) / tpb;
  return (int)(b > 8192 ? 8192 : (b < 1 ? 1 : b));
}

}  // namespace ddit

using namespace ddit;

extern "C" {

DDIT_API int ddit_groupnorm(const void* x, void* y, double* stats, const float* gamma,
                            const float* beta, int N, int P, int C, int G, float eps, int silu_act,
                            void* stream) {
  // `stats` scratch layout: fp64 [N][G][2] followed by the fp32x2 partials [N][nblk][G]
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (C % 8 || C % G || G > 32 || (C / 8) > 256 || 256 % (C / 8)) {
    set_error("groupnorm: C a power of two in [8, 2048] divisible by G <= 32 required");
    return DDIT_E_INVALID;
  }
  int ppb = 1024;
  int nblk = (P + ppb - 1) / ppb;
  if (nblk > 512) {  // bound the partial buffer: larger pixel chunks per block
    ppb = (P + 511) / 512;
    nblk = (P + ppb - 1) / ppb;
  }
  float2* partial = reinterpret_cast<float2*>(stats + (size_t)N * G * 2);
  gn_partial_kernel<<<dim3(nblk, N), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x), partial, P,
                                                  C, G, ppb, nblk);
  gn_finalize_kernel<<<N, 32, 0, s>>>(partial, stats, G, nblk);
  const size_t vecs = (size_t)N * P * (C / 8);
  gn_apply_kernel<<<blocks_for(vecs, 256), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x),
                                                         static_cast<__nv_bfloat16*>(y), stats,
                                                         gamma, beta, P, C, G, eps, silu_act, vecs);
  return check_cuda("groupnorm");
}

DDIT_API int ddit_upsample2x(const void* x, void* y, int N, int H, int W, int C, void* stream) {
  if (C % 8) {
    set_error("upsample2x: C %% 8 required");
    return DDIT_E_INVALID;
  }
  const size_t total = (size_t)N * 4 * H * W * (C / 8);
  upsample2x_kernel<<<blocks_for(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), N, H, W, C);
  return check_cuda("upsample2x");
}

DDIT_API int ddit_depth_to_time(const void* x, void* y, int B, int T, int HW, int C, void* stream) {
  const size_t total = (size_t)B * 2 * T * HW * C;
  depth_to_time_kernel<<<blocks_for(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), B, T, HW, C);
  return check_cuda("depth_to_time");
}

DDIT_API int ddit_conv_small(const void* x, int x_is_f32, const long long* x_strides,
                             const float* w, const float* bias, void* y, int B, int T, int H, int W,
                             int Cin, int Cout, int kt, int kh, int kw, int causal_time, int out_cf,
                             int Hc, int Wc, void* stream) {
  XStrides xs;
  if (x_strides) {
    xs.b = x_strides[0]; xs.c = x_strides[1]; xs.t = x_strides[2]; xs.h = x_strides[3];
    xs.w = x_strides[4];
  } else {  // dense channels-last
    xs.c = 1; xs.w = Cin; xs.h = (long long)W * Cin; xs.t = (long long)H * W * Cin;
    xs.b = (long long)T * H * W * Cin;
  }
  const size_t npix = (size_t)B * T * H * W;
  dim3 block(32, 4);
  const int pt = causal_time ? kt - 1 : kt / 2;
  const int grid = (int)((npix + 3) / 4);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (x_is_f32)
    conv_small_kernel<float><<<grid, block, 0, s>>>(static_cast<const float*>(x), xs, w, bias, y, B,
                                                   T, H, W, Cin, Cout, kt, kh, kw, pt, out_cf, Hc, Wc);
  else
    conv_small_kernel<__nv_bfloat16><<<grid, block, 0, s>>>(
        static_cast<const __nv_bfloat16*>(x), xs, w, bias, y, B, T, H, W, Cin, Cout, kt, kh, kw, pt,
        out_cf, Hc, Wc);
  return check_cuda("conv_small");
}

DDIT_API int ddit_softmax_rows(const float* S, void* P, int rows, int cols, int valid, float scale,
                               void* stream) {
  softmax_rows_kernel<<<rows, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      S, static_cast<__nv_bfloat16*>(P), rows, cols, valid, scale);
  return check_cuda("softmax_rows");
}

DDIT_API int ddit_transpose_bf16(const void* in, void* out, int rows, int cols, int ld_in,
                                 int rows_pad, void* stream) {
  dim3 grid((cols + 31) / 32, (rows_pad + 31) / 32);
  transpose_kernel<<<grid, dim3(32, 8), 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(in), static_cast<__nv_bfloat16*>(out), rows, cols, ld_in,
      rows_pad);
  return check_cuda("transpose");
}

DDIT_API int ddit_add_f32_bf16(const float* a, const void* b, void* y, uint64_t n, void* stream) {
  add_f32_bf16_kernel<<<blocks_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      a, static_cast<const __nv_bfloat16*>(b), static_cast<__nv_bfloat16*>(y), n);
  return check_cuda("add");
}

}  // extern "C"
