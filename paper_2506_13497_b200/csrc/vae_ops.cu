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
// Deterministic two-level statistics (fixed reduction order: bitwise reproducible), then one
// streaming pass:
//   gn_partial:  block (blk, n) reduces pixels [blk*ppb, (blk+1)*ppb) of sample n into
//                partial[n][blk][g] = (sum, sumsq). Thread t owns the 8-channel vector t % (C/8)
//                (C/8 divides 256), walks pixels with stride 256 / (C/8), 4 loads in flight, folds
//                its 8 channels into their group(s) and the G owner threads add the 256/G
//                contributions of their group in a fixed order.
//   gn_finalize: fp64 sum of the partials in block order -> mean / rstd per (n, g) -> per-channel
//                affine coefficients coef[n][c] = (a, b), a = rstd*gamma, b = beta - mean*a.
//   gn_apply:    y = act(x*a + b), one FMA per element (+ SiLU as x*(0.5 + 0.5*tanh(x/2)), one MUFU
//                op); the thread's channel vector is fixed, so its 16 coefficients stay in registers.
constexpr int kGnUnroll = 4;       // vectors in flight per thread, apply
constexpr int kGnPartUnroll = 8;   // statistics: partition granule (pixels per thread)

// The block's pixels [p0, p1) of sample n are one contiguous byte range: it streams through a
// ring of kGnStages 16 KB shared-memory stages filled by bulk async copies (one elected thread,
// mbarrier completion), so ~48 KB per block are in flight without relying on per-thread loads.
constexpr int kGnStageBytes = 16384, kGnStages = 3;
constexpr int kGnPartSmem = kGnStages * kGnStageBytes + kGnStages * 8;

DDIT_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Persistent: block b takes chunks (n, blk) = b, b + gridDim.x, ... of the N x nblk chunks, and its
// ring runs across chunk boundaries (the next chunk's stages load while this one is reduced). A
// chunk's sums do not depend on which block takes it (same per-thread order, same fixed fold).
__global__ void __launch_bounds__(256)
    gn_partial_kernel(const __nv_bfloat16* __restrict__ x, float2* __restrict__ partial, int N,
                      int P, int C, int G, int ppb, int nblk) {
  extern __shared__ __align__(128) uint8_t gn_smem[];
  const int cg = C / G;
  const int vecs = C / 8;
  const int step = 256 / vecs;
  __shared__ float2 red[256][8];
  const uint4* ring = reinterpret_cast<const uint4*>(gn_smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(gn_smem + kGnStages * kGnStageBytes);
  const int nchunks = N * nblk;
  const uint32_t row_bytes = (uint32_t)C * 2;
  auto chunk_bytes = [&](int c) -> uint32_t {
    const int p0 = (c % nblk) * ppb;
    return (uint32_t)(min(p0 + ppb, P) - p0) * row_bytes;
  };
  auto chunk_src = [&](int c) -> const char* {
    return reinterpret_cast<const char*>(x + ((size_t)(c / nblk) * P + (size_t)(c % nblk) * ppb) * C);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < kGnStages; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  // producer cursor (thread 0 only): chunk ic, byte offset ioff, ring slot counter ig
  int ic = blockIdx.x, ig = 0;
  uint32_t ioff = 0;
  auto issue_next = [&]() {
    if (ic >= nchunks) return;
    const uint32_t total = chunk_bytes(ic);
    const uint32_t bytes = min((uint32_t)kGnStageBytes, total - ioff);
    uint64_t* bar = &full[ig % kGnStages];
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s(gn_smem + (ig % kGnStages) * kGnStageBytes, chunk_src(ic) + ioff, bytes, bar);
    ++ig;
    ioff += bytes;
    if (ioff >= total) {
      ioff = 0;
      ic += gridDim.x;
    }
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < kGnStages; ++i) issue_next();
  int g_cons = 0;  // consumer ring counter
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
    float sg[8], qg[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) sg[e] = qg[e] = 0.f;
    const uint32_t total = chunk_bytes(c);
    // stage offsets are multiples of 1024 vectors and 256 of C/8: thread t always sees channel
    // vector t % (C/8)
    for (uint32_t off = 0; off < total; off += kGnStageBytes, ++g_cons) {
      mbar_wait(&full[g_cons % kGnStages], (g_cons / kGnStages) & 1);
      const int nv = (int)(min((uint32_t)kGnStageBytes, total - off) / 16);
      const uint4* sv = ring + (g_cons % kGnStages) * (kGnStageBytes / 16);
      for (int i = threadIdx.x; i < nv; i += 256) {
        const uint4 u = sv[i];
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = unpack_bf16(w[e]);
          sg[2 * e] += f.x;
          sg[2 * e + 1] += f.y;
          qg[2 * e] = fmaf(f.x, f.x, qg[2 * e]);
          qg[2 * e + 1] = fmaf(f.y, f.y, qg[2 * e + 1]);
        }
      }
      __syncthreads();  // stage consumed by every thread: refill its slot
      if (threadIdx.x == 0) issue_next();
    }
    // fold the 8 channels into their group(s): slot j holds group (v*8 + j*cg) / cg
    const int gpv = cg >= 8 ? 1 : 8 / cg;  // groups per 8-channel vector
    const int width = 8 / gpv;
    for (int j = 0; j < gpv; ++j) {
      float s = 0.f, q = 0.f;
      for (int e = j * width; e < (j + 1) * width; ++e) {
        s += sg[e];
        q += qg[e];
      }
      red[threadIdx.x][j] = make_float2(s, q);
    }
    __syncthreads();
    if (threadIdx.x < G) {
      const int g = threadIdx.x;
      float s = 0.f, q = 0.f;
      if (cg >= 8) {
        const int vpg = cg / 8;
        for (int k = 0; k < step; ++k)
          for (int j = 0; j < vpg; ++j) {
            const float2 r = red[k * vecs + g * vpg + j][0];
            s += r.x;
            q += r.y;
          }
      } else {
        for (int k = 0; k < step; ++k) {
          const float2 r = red[k * vecs + g / gpv][g % gpv];
          s += r.x;
          q += r.y;
        }
      }
      // [n][g][blk]: the finalize reads a group's partials as one contiguous run
      partial[((size_t)(c / nblk) * G + g) * nblk + c % nblk] = make_float2(s, q);
    }
    __syncthreads();  // red reused by the next chunk
  }
}

// grid (N, G / 8): one warp per (sample, group); a group's partials are contiguous, so the
// lanes' loads coalesce (the [n][blk][g] layout made them 256 B-strided: 15 us per call on one SM)
__global__ void __launch_bounds__(256)
    gn_finalize_kernel(const float2* __restrict__ partial, float2* __restrict__ coef,
                       const float* __restrict__ gamma, const float* __restrict__ beta, int P,
                       int C, int G, int nblk, float eps) {
  const int n = blockIdx.x;
  __shared__ double mean_s[8], rstd_s[8];
  // lanes take blocks lane, lane+32, ... then a fixed xor tree (deterministic)
  const int lane = threadIdx.x & 31, wg = threadIdx.x >> 5;
  const int g = blockIdx.y * 8 + wg;
  if (g < G) {
    double s = 0, q = 0;
    const float2* pg = partial + ((size_t)n * G + g) * nblk;
    for (int b = lane; b < nblk; b += 32) {
      const float2 v = pg[b];
      s += v.x;
      q += v.y;
    }
    for (int o = 16; o; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      q += __shfl_xor_sync(0xffffffffu, q, o);
    }
    if (lane == 0) {
      const double cnt = (double)P * (C / G);
      const double mean = s / cnt;
      const double var = fmax(q / cnt - mean * mean, 0.0);
      mean_s[wg] = mean;
      rstd_s[wg] = (double)rsqrtf((float)var + eps);
    }
  }
  __syncthreads();
  const int cg = C / G;
  const int c0 = blockIdx.y * 8 * cg, c1 = min(C, c0 + 8 * cg);
  for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    const double a = rstd_s[(c - c0) / cg] * (double)gamma[c];
    coef[(size_t)n * C + c] = make_float2((float)a, (float)((double)beta[c] - mean_s[(c - c0) / cg] * a));
  }
}

DDIT_DEV float silu_fast(float v) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * v));
  return v * fmaf(0.5f, t, 0.5f);
}

// grid (chunks, N); block chunk covers 256*kGnUnroll consecutive 8-channel vectors of sample n
template <bool SILU>
__global__ void __launch_bounds__(256)
    gn_apply_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                    const float2* __restrict__ coef, int C, size_t vecs_per_n) {
  const int n = blockIdx.y;
  const int vecs = C / 8;
  const int v = threadIdx.x % vecs;  // fixed: 256 is a multiple of C/8
  float a[8], b[8];
  {
    const float4* cp = reinterpret_cast<const float4*>(coef + (size_t)n * C + v * 8);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 f = cp[k];
      a[2 * k] = f.x;
      b[2 * k] = f.y;
      a[2 * k + 1] = f.z;
      b[2 * k + 1] = f.w;
    }
  }
  const uint4* src = reinterpret_cast<const uint4*>(x) + (size_t)n * vecs_per_n;
  uint4* dst = reinterpret_cast<uint4*>(y) + (size_t)n * vecs_per_n;
  const size_t i0 = (size_t)blockIdx.x * 256 * kGnUnroll + threadIdx.x;
  uint4 u[kGnUnroll];
#pragma unroll
  for (int k = 0; k < kGnUnroll; ++k) {
    const size_t i = i0 + (size_t)k * 256;
    u[k] = i < vecs_per_n ? __ldcs(src + i) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int k = 0; k < kGnUnroll; ++k) {
    const size_t i = i0 + (size_t)k * 256;
    const uint32_t w[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = unpack_bf16(w[e]);
      float r0 = fmaf(f.x, a[2 * e], b[2 * e]), r1 = fmaf(f.y, a[2 * e + 1], b[2 * e + 1]);
      if (SILU) {
        r0 = silu_fast(r0);
        r1 = silu_fast(r1);
      }
      o[e] = pack_bf16(r0, r1);
    }
    if (i < vecs_per_n) dst[i] = make_uint4(o[0], o[1], o[2], o[3]);
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
// (element strides xs = {b, c, t, h, w}; bf16 or fp32), w: fp32 [kt][kh][kw][Cin][Cout] (lanes
// read consecutive output channels), y: [B][T][H][W][Cout] bf16, or fp32 channels-first
// [B][Cout][T][Hc][Wc] cropped to (Hc, Wc) when out_cf is set. A warp computes kConvSmallPix
// consecutive pixels, lanes over output channels: each weight load feeds kConvSmallPix FMAs,
// the input loads are warp broadcasts.
struct XStrides {
  long long b, c, t, h, w;
};
constexpr int kConvSmallPix = 4;
// COL output channels per lane (lane, lane+32, ...): the tap's input values, loaded once, feed
// kConvSmallPix x COL FMAs
template <typename TIn, int COL>
__global__ void __launch_bounds__(128)
    conv_small_kernel(const TIn* __restrict__ x, XStrides xs, const float* __restrict__ w,
                      const float* __restrict__ bias, void* __restrict__ y, int B, int T, int H,
                      int W, int Cin, int Cout, int kt, int kh, int kw, int pt, int out_cf, int Hc,
                      int Wc) {
  constexpr int NP = kConvSmallPix;
  const size_t npix = (size_t)B * T * H * W;
  const size_t pix0 = ((size_t)blockIdx.x * blockDim.y + threadIdx.y) * NP;
  if (pix0 >= npix) return;
  int bq[NP], tq[NP], yq[NP], xq[NP];
  bool ok[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const size_t pix = pix0 + p;
    ok[p] = pix < npix;
    const size_t q = ok[p] ? pix : pix0;
    xq[p] = (int)(q % W);
    size_t r = q / W;
    yq[p] = (int)(r % H);
    r /= H;
    tq[p] = (int)(r % T);
    bq[p] = (int)(r / T);
  }
  for (int co0 = threadIdx.x; co0 < Cout; co0 += 32 * COL) {
    float acc[NP][COL];
#pragma unroll
    for (int j = 0; j < COL; ++j) {
      const int co = co0 + 32 * j;
      const float b0 = (bias && co < Cout) ? bias[co] : 0.f;
#pragma unroll
      for (int p = 0; p < NP; ++p) acc[p][j] = b0;
    }
    for (int dt = 0; dt < kt; ++dt)
      for (int dy = 0; dy < kh; ++dy)
        for (int dx = 0; dx < kw; ++dx) {
          const TIn* xp[NP];
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            const int ti = tq[p] + dt - pt, yi = yq[p] + dy - kh / 2, xi = xq[p] + dx - kw / 2;
            xp[p] = (ti < 0 || ti >= T || yi < 0 || yi >= H || xi < 0 || xi >= W)
                        ? nullptr
                        : x + bq[p] * xs.b + ti * xs.t + yi * xs.h + xi * xs.w;
          }
          const float* wp = w + (((size_t)dt * kh + dy) * kw + dx) * Cin * Cout + co0;
          for (int ci = 0; ci < Cin; ++ci) {
            float xv[NP];
#pragma unroll
            for (int p = 0; p < NP; ++p) xv[p] = xp[p] ? static_cast<float>(xp[p][ci * xs.c]) : 0.f;
#pragma unroll
            for (int j = 0; j < COL; ++j) {
              const float wv = (co0 + 32 * j < Cout) ? wp[(size_t)ci * Cout + 32 * j] : 0.f;
#pragma unroll
              for (int p = 0; p < NP; ++p) acc[p][j] = fmaf(wv, xv[p], acc[p][j]);
            }
          }
        }
#pragma unroll
    for (int j = 0; j < COL; ++j) {
      const int co = co0 + 32 * j;
      if (co >= Cout) continue;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        if (!ok[p]) continue;
        if (out_cf) {
          if (yq[p] < Hc && xq[p] < Wc)
            static_cast<float*>(y)[((((size_t)bq[p] * Cout + co) * T + tq[p]) * Hc + yq[p]) * Wc + xq[p]] =
                acc[p][j];
        } else {
          static_cast<__nv_bfloat16*>(y)[(pix0 + p) * Cout + co] = __float2bfloat16(acc[p][j]);
        }
      }
    }
  }
}

// decoded frames: channels 0..C-1 of bf16 channels-last y [N][H][W][ld] -> fp32 channels-first
// [C][N][Hc][Wc] (the video tensor [1][C][N][Hc][Wc], cropped); one thread per output pixel, the
// C stores coalesced across threads
__global__ void __launch_bounds__(256)
    frames_out_kernel(const __nv_bfloat16* __restrict__ y, float* __restrict__ out, int N, int H,
                      int W, int ld, int C, int Hc, int Wc) {
  const size_t plane = (size_t)Hc * Wc;
  const size_t total = (size_t)N * plane;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int n = (int)(i / plane);
    const int r = (int)(i % plane);
    const int yy = r / Wc, xx = r % Wc;
    const __nv_bfloat16* src = y + (((size_t)n * H + yy) * W + xx) * ld;
    for (int c = 0; c < C; ++c) out[((size_t)c * N + n) * plane + r] = __bfloat162float(src[c]);
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
  // `stats` scratch layout: fp64 [N][G][2] followed by the fp32x2 partials [N][G][nblk]
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (C % 8 || C % G || G > 32 || (C / 8) > 256 || 256 % (C / 8)) {
    set_error("groupnorm: C a power of two in [8, 2048] divisible by G <= 32 required");
    return DDIT_E_INVALID;
  }
  // >= 1024 pixels per block, but >= 2 blocks per SM of one sample (temporal-VAE calls have
  // N = 1); at most 512 blocks per sample (partial buffer bound). The partition depends on P and C
  // only, never on N: a frame's statistics must not change with how many frames share the call
  // (VAE DoP decodes frame ranges and must reproduce the whole decode bit for bit).
  const int step = 256 / (C / 8);
  int nblk = (P + 1023) / 1024;
  nblk = std::max(nblk, std::min(296, (P + step * kGnPartUnroll - 1) / (step * kGnPartUnroll)));
  nblk = std::max(1, std::min(nblk, 512));
  const int ppb = (P + nblk - 1) / nblk;
  nblk = (P + ppb - 1) / ppb;
  float2* partial = reinterpret_cast<float2*>(stats + (size_t)N * G * 2);
  float2* coef = partial + (size_t)N * nblk * G;
  static size_t attr[64] = {};
  ensure_smem((const void*)gn_partial_kernel, kGnPartSmem, attr);
  static int sms[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  const int pgrid = std::max(1, std::min(N * nblk, 3 * sms[dev]));  // persistent, 3 per SM
  gn_partial_kernel<<<pgrid, 256, kGnPartSmem, s>>>(static_cast<const __nv_bfloat16*>(x), partial, N,
                                                    P, C, G, ppb, nblk);
  gn_finalize_kernel<<<dim3(N, (G + 7) / 8), 256, 0, s>>>(partial, coef, gamma, beta, P, C, G, nblk, eps);
  const size_t vpn = (size_t)P * (C / 8);
  const dim3 grid((unsigned)((vpn + 256 * kGnUnroll - 1) / (256 * kGnUnroll)), N);
  if (silu_act)
    gn_apply_kernel<true><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x),
                                               static_cast<__nv_bfloat16*>(y), coef, C, vpn);
  else
    gn_apply_kernel<false><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x),
                                                static_cast<__nv_bfloat16*>(y), coef, C, vpn);
  return check_cuda("groupnorm");
}

DDIT_API int ddit_groupnorm_partials(const void* x, void* y, const float* partial, int nblk,
                                     float* coef, const float* gamma, const float* beta, int N,
                                     int P, int C, int G, float eps, int silu_act, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (C % 8 || C % G || G > 32 || (C / 8) > 256 || 256 % (C / 8) || nblk < 1) {
    set_error("groupnorm_partials: C a power of two in [8, 2048] divisible by G <= 32, nblk >= 1");
    return DDIT_E_INVALID;
  }
  float2* cf = reinterpret_cast<float2*>(coef);
  gn_finalize_kernel<<<dim3(N, (G + 7) / 8), 256, 0, s>>>(reinterpret_cast<const float2*>(partial), cf,
                                                          gamma, beta, P, C, G, nblk, eps);
  const size_t vpn = (size_t)P * (C / 8);
  const dim3 grid((unsigned)((vpn + 256 * kGnUnroll - 1) / (256 * kGnUnroll)), N);
  if (silu_act)
    gn_apply_kernel<true><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x),
                                               static_cast<__nv_bfloat16*>(y), cf, C, vpn);
  else
    gn_apply_kernel<false><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x),
                                                static_cast<__nv_bfloat16*>(y), cf, C, vpn);
  return check_cuda("groupnorm_partials");
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
  const int grid = (int)((npix + 4 * kConvSmallPix - 1) / (4 * kConvSmallPix));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool wide = Cout % 128 == 0;
#define DDIT_CONV_SMALL(TIN, COL)                                                              \
  conv_small_kernel<TIN, COL><<<grid, block, 0, s>>>(static_cast<const TIN*>(x), xs, w, bias, y, B, \
                                                     T, H, W, Cin, Cout, kt, kh, kw, pt, out_cf, Hc, Wc)
  if (x_is_f32) {
    if (wide) DDIT_CONV_SMALL(float, 4); else DDIT_CONV_SMALL(float, 1);
  } else {
    if (wide) DDIT_CONV_SMALL(__nv_bfloat16, 4); else DDIT_CONV_SMALL(__nv_bfloat16, 1);
  }
#undef DDIT_CONV_SMALL
  return check_cuda("conv_small");
}

DDIT_API int ddit_frames_out(const void* y, float* out, int N, int H, int W, int ld, int C, int Hc,
                             int Wc, void* stream) {
  if (C > ld || Hc > H || Wc > W) {
    set_error("frames_out: crop larger than the source");
    return DDIT_E_INVALID;
  }
  frames_out_kernel<<<blocks_for((size_t)N * Hc * Wc, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(y), out, N, H, W, ld, C, Hc, Wc);
  return check_cuda("frames_out");
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
