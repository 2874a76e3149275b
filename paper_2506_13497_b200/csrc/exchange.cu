// DSP all-to-all between the spatial (T-sharded) and temporal (S-sharded) layouts
// (SURVEY.md §2.3 K8 / §8(a) n3, n5), pushed as direct stores into every destination
// rank's buffer (peer pointers over NVLink, or local buffers for virtual ranks), plus a
// flag barrier across ranks.
//
//   x_sp of rank r: [B][Tl_r][S][C]      (frames t_lo_r .. t_lo_r + Tl_r - 1, all tokens)
//   x_tp of rank q: [B][T][Sl_q][C]      (all frames, tokens s_lo_q .. s_lo_q + Sl_q - 1)
// One warp moves one token row (C fp32) with 16-byte vectors.
#include "common.cuh"
#include "exchange.cuh"

namespace ddit {

__global__ void __launch_bounds__(256)
    exchange_sp_to_tp_kernel(const float* __restrict__ src, PeerPtrs dst, int B, int T, int S,
                             int C, int P, int t_lo, int Tl, int s_chunk) {
  const int rows = B * Tl * S;
  const int nv = C >> 2;
  for (int row = blockIdx.x * 8 + (threadIdx.x >> 5); row < rows; row += gridDim.x * 8) {
    const int s = row % S;
    const int tl = (row / S) % Tl;
    const int b = row / (S * Tl);
    const int q = s / s_chunk;
    const int s_lo = q * s_chunk;
    const int s_hi = min(s_lo + s_chunk, S);
    const int Sl = s_hi - s_lo;
    const float4* sp = reinterpret_cast<const float4*>(src + (size_t)row * C);
    float4* dp = reinterpret_cast<float4*>(dst.p[q] +
                                           (((size_t)b * T + t_lo + tl) * Sl + (s - s_lo)) * C);
    for (int i = threadIdx.x & 31; i < nv; i += 32) dp[i] = __ldg(sp + i);
  }
}

__global__ void __launch_bounds__(256)
    exchange_tp_to_sp_kernel(const float* __restrict__ src, PeerPtrs dst, int B, int T, int S,
                             int C, int P, int s_lo, int Sl, int t_chunk) {
  const int rows = B * T * Sl;
  const int nv = C >> 2;
  for (int row = blockIdx.x * 8 + (threadIdx.x >> 5); row < rows; row += gridDim.x * 8) {
    const int sl = row % Sl;
    const int t = (row / Sl) % T;
    const int b = row / (Sl * T);
    const int q = t / t_chunk;
    const int t_lo = q * t_chunk;
    const int t_hi = min(t_lo + t_chunk, T);
    const int Tlq = t_hi - t_lo;
    const float4* sp = reinterpret_cast<const float4*>(src + (size_t)row * C);
    float4* dp = reinterpret_cast<float4*>(dst.p[q] +
                                           (((size_t)b * Tlq + (t - t_lo)) * S + s_lo + sl) * C);
    for (int i = threadIdx.x & 31; i < nv; i += 32) dp[i] = __ldg(sp + i);
  }
}

int exchange_sp_to_tp(const float* src, const PeerPtrs& dst, int B, int T, int S, int C, int P,
                      int t_lo, int Tl, cudaStream_t s) {
  const int rows = B * Tl * S;
  if (rows <= 0) return 0;
  const int s_chunk = (S + P - 1) / P;
  int grid = (rows + 7) / 8;
  if (grid > 4 * 148) grid = 4 * 148;
  exchange_sp_to_tp_kernel<<<grid, 256, 0, s>>>(src, dst, B, T, S, C, P, t_lo, Tl, s_chunk);
  return 0;
}

int exchange_tp_to_sp(const float* src, const PeerPtrs& dst, int B, int T, int S, int C, int P,
                      int s_lo, int Sl, cudaStream_t s) {
  const int rows = B * T * Sl;
  if (rows <= 0) return 0;
  const int t_chunk = (T + P - 1) / P;
  int grid = (rows + 7) / 8;
  if (grid > 4 * 148) grid = 4 * 148;
  exchange_tp_to_sp_kernel<<<grid, 256, 0, s>>>(src, dst, B, T, S, C, P, s_lo, Sl, t_chunk);
  return 0;
}

// Flag barrier: thread q publishes `epoch` into rank q's flag slot for this rank, then every
// thread waits until its own slot from rank q reached `epoch`. Flags live in memory visible to
// all ranks (peer-mapped); system-scope release/acquire orders the pushed rows.
__global__ void flag_barrier_kernel(PeerFlags flags, int rank, int P, uint32_t epoch) {
  const int q = threadIdx.x;
  if (q >= P) return;
  __threadfence_system();
  volatile uint32_t* remote = flags.p[q] + rank;
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(remote), "r"(epoch) : "memory");
  volatile uint32_t* mine = flags.p[rank] + q;
  uint32_t v;
  do {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
  } while ((int32_t)(v - epoch) < 0);
}

int flag_barrier(const PeerFlags& flags, int rank, int P, uint32_t epoch, cudaStream_t s) {
  flag_barrier_kernel<<<1, 32, 0, s>>>(flags, rank, P, epoch);
  return 0;
}

}  // namespace ddit
