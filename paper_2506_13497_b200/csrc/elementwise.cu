// Memory-bound kernels of the STDiT3 step: fused
// LayerNorm + t2i-modulate, timestep / fps embedding GEMVs, the per-step modulation table of
// all blocks, patch-embed + pos-embed (step entry), and the fused exit (final LayerNorm +
// modulate + Linear + unpatchify + CFG combine + rectified-flow Euler update).
#include "common.cuh"
#include <cstdlib>
#include "elementwise.cuh"

namespace ddit {

// ------------------------------------------------------------------ LN + modulate (K1)
// xm[r, :] = bf16( LN(x[r, :]) * (1 + scale[b]) + shift[b] ),  b = r / rows_per_b.
// LPR lanes per row, NV float4 per lane (the whole row in registers, C = 4 * LPR * NV exactly
// for the instantiated widths, else the generic NV = kMaxVec path with bounds checks): two-pass
// statistics from registers, x streamed once (__ldcs), shift / scale through L1.
static constexpr int kMaxVec = 12;  // generic path: C up to 1536 with 32 lanes

template <int LPR>
DDIT_DEV float group_sum(float v) {
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NV, int LPR, bool EXACT>
__global__ void __launch_bounds__(128)
    ln_modulate_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ out, int M, int C,
                       const float* __restrict__ shift, const float* __restrict__ scale,
                       int mod_stride, int rows_per_b, float eps) {
  pdl_wait();
  constexpr int RPB = 128 / LPR;  // rows per block
  const int row = blockIdx.x * RPB + (threadIdx.x / LPR);
  const int lane = threadIdx.x % LPR;
  const bool live = row < M;  // all lanes of a warp take part in the shuffles
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)(live ? row : 0) * C);
  const int nv = C >> 2;
  float4 v[NV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + LPR * i;
    if (live && (EXACT || c < nv)) {
      v[i] = __ldcs(xr + c);
      s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
  }
  const float mean = group_sum<LPR>(s) / C;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + LPR * i;
    if (live && (EXACT || c < nv)) {
      const float a = v[i].x - mean, b = v[i].y - mean, cc = v[i].z - mean, d = v[i].w - mean;
      q += (a * a + b * b) + (cc * cc + d * d);
    }
  }
  const float rstd = rsqrtf(group_sum<LPR>(q) / C + eps);
  if (!live) return;
  const int bidx = row / rows_per_b;
  const float4* sh = reinterpret_cast<const float4*>(shift + (size_t)bidx * mod_stride);
  const float4* sc = reinterpret_cast<const float4*>(scale + (size_t)bidx * mod_stride);
  uint2* o = reinterpret_cast<uint2*>(out + (size_t)row * C);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + LPR * i;
    if (EXACT || c < nv) {
      const float4 a = __ldg(sh + c), k = __ldg(sc + c);
      const float y0 = (v[i].x - mean) * rstd * (1.f + k.x) + a.x;
      const float y1 = (v[i].y - mean) * rstd * (1.f + k.y) + a.y;
      const float y2 = (v[i].z - mean) * rstd * (1.f + k.z) + a.z;
      const float y3 = (v[i].w - mean) * rstd * (1.f + k.w) + a.w;
      o[c] = make_uint2(pack_bf16(y0, y1), pack_bf16(y2, y3));
    }
  }
}

// C = 1152 streaming variant: a persistent grid of warps, each walking rows r, r + nwarps, ...
// with the NEXT row's 9 float4 per lane loaded before the current row's reductions and stores,
// so every warp keeps a row of loads in flight across its whole life (no block-launch tails).
__global__ void __launch_bounds__(256)
    ln_modulate_stream_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ out, int M,
                              const float* __restrict__ shift, const float* __restrict__ scale,
                              int mod_stride, int rows_per_b, float eps) {
  constexpr int C = 1152, NV = 9;
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * (blockDim.x >> 5);
  int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= M) return;
  float4 v[NV];
  {
    const float4* xr = reinterpret_cast<const float4*>(x + (size_t)row * C);
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = __ldcs(xr + lane + 32 * i);
  }
  for (;;) {
    const int next = row + nw;
    float4 nx[NV];
    if (next < M) {
      const float4* xr = reinterpret_cast<const float4*>(x + (size_t)next * C);
#pragma unroll
      for (int i = 0; i < NV; ++i) nx[i] = __ldcs(xr + lane + 32 * i);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    const float mean = group_sum<32>(s) * (1.f / C);
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float a = v[i].x - mean, b = v[i].y - mean, cc = v[i].z - mean, d = v[i].w - mean;
      q += (a * a + b * b) + (cc * cc + d * d);
    }
    const float rstd = rsqrtf(group_sum<32>(q) * (1.f / C) + eps);
    const int bidx = row / rows_per_b;
    const float4* sh = reinterpret_cast<const float4*>(shift + (size_t)bidx * mod_stride);
    const float4* sc = reinterpret_cast<const float4*>(scale + (size_t)bidx * mod_stride);
    uint2* o = reinterpret_cast<uint2*>(out + (size_t)row * C);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + 32 * i;
      const float4 a = __ldg(sh + c), k = __ldg(sc + c);
      const float y0 = (v[i].x - mean) * rstd * (1.f + k.x) + a.x;
      const float y1 = (v[i].y - mean) * rstd * (1.f + k.y) + a.y;
      const float y2 = (v[i].z - mean) * rstd * (1.f + k.z) + a.z;
      const float y3 = (v[i].w - mean) * rstd * (1.f + k.w) + a.w;
      o[c] = make_uint2(pack_bf16(y0, y1), pack_bf16(y2, y3));
    }
    if (next >= M) break;
    row = next;
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = nx[i];
  }
}

// Variant 5: the streaming kernel with the row's modulation (shift, scale: 18 float4 per lane)
// held in registers and reloaded only when the warp's batch index changes, so a row costs the
// L1 4.6 KB of x + 2.3 KB of stores instead of + 9.2 KB of modulation loads. Same arithmetic.
__global__ void __launch_bounds__(128)
    ln_modulate_stream_regmod_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ out,
                                     int M, const float* __restrict__ shift,
                                     const float* __restrict__ scale, int mod_stride,
                                     int rows_per_b, float eps) {
  constexpr int C = 1152, NV = 9;
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * (blockDim.x >> 5);
  int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= M) return;
  float4 v[NV], sh[NV], sc[NV];
  int cur_b = -1;
  {
    const float4* xr = reinterpret_cast<const float4*>(x + (size_t)row * C);
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = __ldcs(xr + lane + 32 * i);
  }
  for (;;) {
    const int next = row + nw;
    float4 nx[NV];
    if (next < M) {
      const float4* xr = reinterpret_cast<const float4*>(x + (size_t)next * C);
#pragma unroll
      for (int i = 0; i < NV; ++i) nx[i] = __ldcs(xr + lane + 32 * i);
    }
    const int bidx = row / rows_per_b;
    if (bidx != cur_b) {
      cur_b = bidx;
      const float4* a = reinterpret_cast<const float4*>(shift + (size_t)bidx * mod_stride);
      const float4* k = reinterpret_cast<const float4*>(scale + (size_t)bidx * mod_stride);
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        sh[i] = __ldg(a + lane + 32 * i);
        sc[i] = __ldg(k + lane + 32 * i);
      }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    const float mean = group_sum<32>(s) * (1.f / C);
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float a = v[i].x - mean, b = v[i].y - mean, cc = v[i].z - mean, d = v[i].w - mean;
      q += (a * a + b * b) + (cc * cc + d * d);
    }
    const float rstd = rsqrtf(group_sum<32>(q) * (1.f / C) + eps);
    uint2* o = reinterpret_cast<uint2*>(out + (size_t)row * C);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float y0 = (v[i].x - mean) * rstd * (1.f + sc[i].x) + sh[i].x;
      const float y1 = (v[i].y - mean) * rstd * (1.f + sc[i].y) + sh[i].y;
      const float y2 = (v[i].z - mean) * rstd * (1.f + sc[i].z) + sh[i].z;
      const float y3 = (v[i].w - mean) * rstd * (1.f + sc[i].w) + sh[i].w;
      o[lane + 32 * i] = make_uint2(pack_bf16(y0, y1), pack_bf16(y2, y3));
    }
    if (next >= M) break;
    row = next;
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = nx[i];
  }
}

static int g_ln_variant = -1;  // tuning hook (env DDIT_LN): 0 generic, 1 = 32 lanes x 9, 2 = 16 x 18,
                               // 3 = persistent streaming warps (240p: 11.3 / 14.2 us hot / cold),
                               // 5 (default) = 3 with the modulation in registers (9.3 / 12.2 us;
                               // scripts/ln_bench.py, profiles/r02_ln_regmod_bench.txt)

void set_ln_variant(int v) { g_ln_variant = v; }

int ln_modulate(const float* x, __nv_bfloat16* out, int M, int C, const float* shift,
                const float* scale, int mod_stride, int rows_per_b, float eps, cudaStream_t s) {
  if (C % 4 || C > 32 * 4 * kMaxVec || M <= 0) return -2;
  if (g_ln_variant < 0) {
    const char* e = getenv("DDIT_LN");
    g_ln_variant = e ? atoi(e) : 5;
  }
  const int rpb = rows_per_b > 0 ? rows_per_b : M;
  if (C == 1152 && g_ln_variant == 3) {
    static int grid_cap = 0;
    if (!grid_cap) {
      int dev = 0, sms = 148, bps = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, ln_modulate_stream_kernel, 256, 0);
      const char* e = getenv("DDIT_LN_BPS");
      if (e && atoi(e) > 0 && atoi(e) < bps) bps = atoi(e);
      grid_cap = sms * (bps > 0 ? bps : 1);
    }
    const int need = (M + 7) / 8;
    launch_pdl(ln_modulate_stream_kernel, dim3(need < grid_cap ? need : grid_cap), dim3(256), 0, s,
               x, out, M, shift, scale, mod_stride, rpb, eps);
  } else if (C == 1152 && g_ln_variant == 5) {
    static int grid_cap = 0;
    if (!grid_cap) {
      int dev = 0, sms = 148, bps = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, ln_modulate_stream_regmod_kernel, 128, 0);
      grid_cap = sms * (bps > 0 ? bps : 1);
    }
    const int need = (M + 3) / 4;
    launch_pdl(ln_modulate_stream_regmod_kernel, dim3(need < grid_cap ? need : grid_cap), dim3(128),
               0, s, x, out, M, shift, scale, mod_stride, rpb, eps);
  } else if (C == 1152 && g_ln_variant == 1) {
    launch_pdl(ln_modulate_kernel<9, 32, true>, dim3((M + 3) / 4), dim3(128), 0, s, x, out, M, C,
               shift, scale, mod_stride, rpb, eps);
  } else if (C == 1152 && g_ln_variant == 2) {
    launch_pdl(ln_modulate_kernel<18, 16, true>, dim3((M + 7) / 8), dim3(128), 0, s, x, out, M, C,
               shift, scale, mod_stride, rpb, eps);
  } else {
    launch_pdl(ln_modulate_kernel<kMaxVec, 32, false>, dim3((M + 3) / 4), dim3(128), 0, s, x, out,
               M, C, shift, scale, mod_stride, rpb, eps);
  }
  return 0;
}

// ------------------------------------------------------------------ t / fps embedding (K10)
// freq[j, :] = [cos(t_j * f), sin(t_j * f)], f_i = exp(-ln(10000) i / half), for the B
// timesteps followed by the B fps values.
__global__ void timestep_freq_kernel(float* __restrict__ freq, const float* __restrict__ tvals,
                                     int nvals, int dim) {
  const int j = blockIdx.x;
  const int half = dim / 2;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const float f = expf(-9.210340371976184f * (float)i / (float)half);  // ln(10000)
    const float a = tvals[j] * f;
    freq[j * dim + i] = cosf(a);
    freq[j * dim + half + i] = sinf(a);
  }
}

// y[b, n] (+)= W[n, :] . act(x[b, :]) + bias[n] ; W bf16 [N, K]; one warp per output n.
// in_act: 0 none, 1 SiLU. out_act: 0 none, 1 SiLU. accumulate: add to y instead of store.
__global__ void __launch_bounds__(256)
    gemv_kernel(const __nv_bfloat16* __restrict__ W, const float* __restrict__ bias,
                const float* __restrict__ x, float* __restrict__ y, int nb, int N, int K,
                int in_act, int out_act, int accumulate) {
  const int n = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (n >= N) return;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const __nv_bfloat16* w = W + (size_t)n * K;
  for (int k = lane * 8; k < K; k += 32 * 8) {
    const uint4 wv = *reinterpret_cast<const uint4*>(w + k);
    const uint32_t wr[4] = {wv.x, wv.y, wv.z, wv.w};
    float wf[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = unpack_bf16(wr[e]);
      wf[2 * e] = f.x;
      wf[2 * e + 1] = f.y;
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (b >= nb) break;
      const float* xb = x + (size_t)b * K + k;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float xv = xb[e];
        if (in_act == 1) xv = silu(xv);
        acc[b] += wf[e] * xv;
      }
    }
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    if (b >= nb) break;
    float r = warp_sum(acc[b]);
    if (lane == 0) {
      r += bias ? bias[n] : 0.f;
      if (out_act == 1) r = silu(r);
      float* dst = y + (size_t)b * N + n;
      *dst = accumulate ? *dst + r : r;
    }
  }
}

int gemv(const __nv_bfloat16* W, const float* bias, const float* x, float* y, int nb, int N, int K,
         int in_act, int out_act, int accumulate, cudaStream_t s) {
  if (nb > 4 || K % 8) return -2;
  gemv_kernel<<<(N + 7) / 8, 256, 0, s>>>(W, bias, x, y, nb, N, K, in_act, out_act, accumulate);
  return 0;
}

int timestep_freq(float* freq, const float* tvals, int nvals, int dim, cudaStream_t s) {
  timestep_freq_kernel<<<nvals, 128, 0, s>>>(freq, tvals, nvals, dim);
  return 0;
}

// mods[blk][b][6C] = sst[blk][6C] + t_mlp[b][6C]   for blk < nblocks
// fin[b][2C]      = fsst[2C] + t[b][C] (broadcast over the 2 rows)
__global__ void modulation_kernel(float* __restrict__ mods, const float* const* __restrict__ sst,
                                  const float* __restrict__ t_mlp, int nblocks, int nb, int C6,
                                  float* __restrict__ fin, const float* __restrict__ fsst,
                                  const float* __restrict__ t, int C) {
  const int blk = blockIdx.y;
  if (blk < nblocks) {
    const float* table = sst[blk];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nb * C6; i += gridDim.x * blockDim.x) {
      const int b = i / C6, j = i % C6;
      mods[((size_t)blk * nb + b) * C6 + j] = table[j] + t_mlp[(size_t)b * C6 + j];
    }
  } else {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nb * 2 * C; i += gridDim.x * blockDim.x) {
      const int b = i / (2 * C), j = i % (2 * C);
      fin[i] = fsst[j] + t[(size_t)b * C + (j % C)];
    }
  }
}

int modulation(float* mods, const float* const* sst, const float* t_mlp, int nblocks, int nb,
               int C, float* fin, const float* fsst, const float* t, cudaStream_t s) {
  dim3 grid(8, nblocks + 1);
  modulation_kernel<<<grid, 256, 0, s>>>(mods, sst, t_mlp, nblocks, nb, 6 * C, fin, fsst, t, C);
  return 0;
}

// ------------------------------------------------------------------ tables
// pos[s][C]: OpenSora PositionEmbedding2D -- first half encodes the column coordinate,
// second half the row coordinate; each half = [sin(p f), cos(p f)], f_i = 10000^(-2i/(C/2)).
__global__ void pos_embed_kernel(float* __restrict__ pos, int h, int w, int C, float scale,
                                 float base_size) {
  const int s = blockIdx.x;
  const int i = s / w, j = s % w;
  const float prow = (float)i / scale * (base_size / (float)h);
  const float pcol = (float)j / scale * (base_size / (float)w);
  const int half = C / 2, q = C / 4;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const int part = c / half;  // 0: column coordinate, 1: row coordinate
    const int r = c % half;
    const int fi = r % q;
    const float f = 1.0f / powf(10000.0f, (float)(2 * fi) / (float)half);
    const float p = (part == 0 ? pcol : prow) * f;
    pos[(size_t)s * C + c] = r < q ? sinf(p) : cosf(p);
  }
}

// rope[t][i] = (cos(t th_i), sin(t th_i)), th_i = 10000^(-2i/D)
__global__ void rope_table_kernel(float2* __restrict__ tab, int T, int D) {
  const int t = blockIdx.x;
  for (int i = threadIdx.x; i < D / 2; i += blockDim.x) {
    const double th = 1.0 / pow(10000.0, (double)(2 * i) / (double)D);
    const double a = (double)t * th;
    tab[t * (D / 2) + i] = make_float2((float)cos(a), (float)sin(a));
  }
}

int build_tables(float* pos, int h, int w, int C, float scale, float base_size, float* rope, int T,
                 int D, cudaStream_t s) {
  pos_embed_kernel<<<h * w, 128, 0, s>>>(pos, h, w, C, scale, base_size);
  rope_table_kernel<<<T, 64, 0, s>>>(reinterpret_cast<float2*>(rope), T, D);
  return 0;
}

// ------------------------------------------------------------------ step entry (K9)
// x[b][t][s][c] = bias[c] + sum_{ci,dh,dw} Wp[c][ci][dh][dw] z[ci][t][2i+dh][2j+dw] + pos[s][c]
// z: the local T-shard [Cin][Tl][Hl][Wl] fp32 (zero outside Hl x Wl); same x for all nb copies.
// One thread per output channel c (its K <= 16 weights in registers), a block per 128 channels x
// 32 tokens: the token patches are staged in smem once per block, the pos-embed row and the
// output row are coalesced over c. (One block per token re-read all C x K weights per token.)
namespace pe {
constexpr int CPB = 128, TPB = 32;
}

__global__ void __launch_bounds__(pe::CPB)
    patch_embed_kernel(const float* __restrict__ z, const float* __restrict__ Wp,
                       const float* __restrict__ bp, const float* __restrict__ pos,
                       float* __restrict__ x, int Tl, int Hl, int Wl, int h, int w, int C,
                       int Cin, int nb) {
  const int S = h * w, ntok = Tl * S, K = Cin * 4;
  const int c = blockIdx.x * pe::CPB + threadIdx.x;
  const int tok0 = blockIdx.y * pe::TPB;
  __shared__ float patch[pe::TPB][16];
  for (int e = threadIdx.x; e < pe::TPB * K; e += pe::CPB) {
    const int tt = e / K, k = e % K, tok = tok0 + tt;
    float v = 0.f;
    if (tok < ntok) {
      const int t = tok / S, sidx = tok % S, i = sidx / w, j = sidx % w;
      const int ci = k / 4, y = 2 * i + (k / 2) % 2, xx = 2 * j + k % 2;
      if (y < Hl && xx < Wl) v = z[(((size_t)ci * Tl + t) * Hl + y) * Wl + xx];
    }
    patch[tt][k] = v;
  }
  __syncthreads();
  if (c >= C) return;
  float wv[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) wv[k] = k < K ? Wp[(size_t)c * K + k] : 0.f;
  const float bias = bp[c];
  for (int tt = 0; tt < pe::TPB; ++tt) {
    const int tok = tok0 + tt;
    if (tok >= ntok) break;
    float acc = bias + pos[(size_t)(tok % S) * C + c];
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < K) acc += wv[k] * patch[tt][k];
    for (int b = 0; b < nb; ++b) x[((size_t)b * Tl * S + tok) * C + c] = acc;
  }
}

int patch_embed(const float* z, const float* Wp, const float* bp, const float* pos, float* x, int Tl,
                int Hl, int Wl, int h, int w, int C, int Cin, int nb, cudaStream_t s) {
  if (Tl <= 0) return 0;
  if (Cin * 4 > 16) return -2;
  const dim3 grid((C + pe::CPB - 1) / pe::CPB, (Tl * h * w + pe::TPB - 1) / pe::TPB);
  patch_embed_kernel<<<grid, pe::CPB, 0, s>>>(z, Wp, bp, pos, x, Tl, Hl, Wl, h, w, C, Cin, nb);
  return 0;
}

// ------------------------------------------------------------------ step exit (K9)
// For each local token (t, s) and both CFG halves b = 0 (cond), 1 (uncond):
//   y_b = LN(x_b) * (1 + scale_b) + shift_b ;  o_b[f] = Wf[f] . y_b + bf[f]
// for the 16 features f = (hp*2 + wp)*out_ch + c with c < Cin (the sigma half is unused);
//   v = o_uncond + g (o_cond - o_uncond);  z[c][t][2i+hp][2j+wp] += v * dt.
// Persistent CTAs keep the 16 used rows of Wf and both rows of the final modulation in smem;
// one warp per token (its two rows in registers, float4 loads). (A CTA per token re-read the
// 74 KB of Wf rows from L2 for every token.)
namespace fl {
constexpr int WARPS = 8, MAXV = 12;  // C <= 32 * 4 * MAXV
}

__global__ void __launch_bounds__(fl::WARPS * 32)
    final_layer_kernel(const float* __restrict__ x, const float* __restrict__ fin,
                       const float* __restrict__ Wf, const float* __restrict__ bf,
                       float* __restrict__ z, int Tl, int Hl, int Wl, int h, int w, int C,
                       int Cin, int out_ch, float guidance, float dt, float eps) {
  extern __shared__ __align__(16) float fl_smem[];
  const int nf = 4 * Cin;                   // used features (<= 16)
  float* wsm = fl_smem;                     // [nf][C]
  float* msm = fl_smem + (size_t)nf * C;    // [2 b][shift C, scale C]
  for (int e = threadIdx.x; e < nf * C; e += blockDim.x) {
    const int f16 = e / C, cc = e % C;
    wsm[e] = Wf[(size_t)((f16 / Cin) * out_ch + f16 % Cin) * C + cc];
  }
  for (int e = threadIdx.x; e < 4 * C; e += blockDim.x) msm[e] = fin[e];
  __syncthreads();
  const int S = h * w, ntok = Tl * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nv = C >> 2;
  for (int tok = blockIdx.x * fl::WARPS + warp; tok < ntok; tok += gridDim.x * fl::WARPS) {
    float o[2];  // this lane's feature ((lane >> 1) & 15) for the two CFG rows
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const float4* xr = reinterpret_cast<const float4*>(x + ((size_t)b * Tl * S + tok) * C);
      float4 v[fl::MAXV];
      float sm = 0.f, sq = 0.f;
#pragma unroll
      for (int k = 0; k < fl::MAXV; ++k) {
        const int q = lane + 32 * k;
        if (q < nv) {
          v[k] = __ldcs(xr + q);
          sm += (v[k].x + v[k].y) + (v[k].z + v[k].w);
          sq += (v[k].x * v[k].x + v[k].y * v[k].y) + (v[k].z * v[k].z + v[k].w * v[k].w);
        }
      }
      sm = warp_sum(sm);
      sq = warp_sum(sq);
      const float mean = sm / C;
      const float rstd = rsqrtf(fmaxf(sq / C - mean * mean, 0.f) + eps);
      const float4* sh = reinterpret_cast<const float4*>(msm + (size_t)b * 2 * C);
      const float4* sc = reinterpret_cast<const float4*>(msm + (size_t)b * 2 * C + C);
#pragma unroll
      for (int k = 0; k < fl::MAXV; ++k) {
        const int q = lane + 32 * k;
        if (q < nv) {
          const float4 a = sh[q], g = sc[q];
          v[k].x = (v[k].x - mean) * rstd * (1.f + g.x) + a.x;
          v[k].y = (v[k].y - mean) * rstd * (1.f + g.y) + a.y;
          v[k].z = (v[k].z - mean) * rstd * (1.f + g.z) + a.z;
          v[k].w = (v[k].w - mean) * rstd * (1.f + g.w) + a.w;
        }
      }
      float part[16];
#pragma unroll
      for (int f = 0; f < 16; ++f) {
        part[f] = 0.f;
        if (f >= nf) continue;
        const float4* wr = reinterpret_cast<const float4*>(wsm + (size_t)f * C);
#pragma unroll
        for (int k = 0; k < fl::MAXV; ++k) {
          const int q = lane + 32 * k;
          if (q < nv) {
            const float4 ww = wr[q];
            part[f] += (v[k].x * ww.x + v[k].y * ww.y) + (v[k].z * ww.z + v[k].w * ww.w);
          }
        }
      }
      // reduce-scatter of the 16 partial sums over the warp: 8 + 4 + 2 + 1 shuffles leave lane l
      // with feature f(l) = bits 4..1 of l summed over 16 lanes, one more shuffle completes it
#pragma unroll
      for (int hbit = 8; hbit >= 1; hbit >>= 1) {
        const bool up = lane & (2 * hbit);
#pragma unroll
        for (int i = 0; i < hbit; ++i) {
          const float send = up ? part[i] : part[i + hbit];
          const float keep = up ? part[i + hbit] : part[i];
          part[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * hbit);
        }
      }
      o[b] = part[0] + __shfl_xor_sync(0xffffffffu, part[0], 1);
    }
    const int t = tok / S, sidx = tok % S, i = sidx / w, j = sidx % w;
    const int f = (lane >> 1) & 15;
    if ((lane & 1) == 0 && f < nf) {
      const int pidx = f / Cin, c = f % Cin;
      const int feat = pidx * out_ch + c;
      const int yy = 2 * i + pidx / 2, xx = 2 * j + pidx % 2;
      if (yy < Hl && xx < Wl) {
        const float oc = o[0] + bf[feat], ou = o[1] + bf[feat];
        const float vv = ou + guidance * (oc - ou);
        float* zp = z + (((size_t)c * Tl + t) * Hl + yy) * Wl + xx;
        *zp = *zp + vv * dt;
      }
    }
  }
}

int final_layer(const float* x, const float* fin, const float* Wf, const float* bf, float* z, int Tl,
                int Hl, int Wl, int h, int w, int C, int Cin, int out_ch, float guidance, float dt,
                float eps, cudaStream_t s) {
  if (Tl <= 0) return 0;
  if (4 * Cin > 16 || C % 4 || C > 32 * 4 * fl::MAXV) return -2;
  const size_t smem = ((size_t)4 * Cin * C + 4 * C) * sizeof(float);
  static size_t attr[64] = {};
  ensure_smem((const void*)final_layer_kernel, smem, attr);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ntok = Tl * h * w;
  const int blocks = (ntok + fl::WARPS - 1) / fl::WARPS;
  final_layer_kernel<<<blocks < 2 * sms ? blocks : 2 * sms, fl::WARPS * 32, smem, s>>>(
      x, fin, Wf, bf, z, Tl, Hl, Wl, h, w, C, Cin, out_ch, guidance, dt, eps);
  return 0;
}

// ------------------------------------------------------------------ misc
__global__ void cast_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                 size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16(in[i]);
}

int cast_bf16(const float* in, __nv_bfloat16* out, size_t n, cudaStream_t s) {
  const int blocks = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  cast_bf16_kernel<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(in, out, n);
  return 0;
}

}  // namespace ddit
