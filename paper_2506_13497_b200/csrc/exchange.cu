// DSP all-to-all between the spatial (T-sharded) and temporal (S-sharded) layouts
// (SURVEY.md §2.3 K8 / §8(a) n3, n5), pushed as direct stores into every destination
// rank's buffer (peer pointers over NVLink, or local buffers for virtual ranks), plus a
// flag barrier across ranks.
//
//   x_sp of rank r: [B][Tl_r][S][C]      (frames t_lo_r .. t_lo_r + Tl_r - 1, all tokens)
//   x_tp of rank q: [B][T][Sl_q][C]      (all frames, tokens s_lo_q .. s_lo_q + Sl_q - 1)
// One warp moves one token row (C fp32) with 16-byte vectors. When flags are registered the
// last CTA to finish (ticket counter) publishes `epoch` into every peer's flag slot for this
// rank after a system-scope fence, so a peer that observes the flag also observes the rows.
#include "common.cuh"
#include "exchange.cuh"

#include <cstdlib>

namespace ddit {

DDIT_DEV void signal_peers(const ExchangeSync& sync) {
  // called by one thread of the last CTA
  __threadfence_system();
  const uint32_t e = *sync.epoch + 1;
  *sync.epoch = e;
  for (int q = 0; q < sync.P; ++q) {
    uint32_t* remote = sync.flags.p[q] + sync.rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(remote), "r"(e) : "memory");
  }
}

DDIT_DEV void finish_cta(const ExchangeSync& sync) {
  if (sync.flags.p[0] == nullptr) return;
  __syncthreads();
  __shared__ unsigned int ticket;
  if (threadIdx.x == 0) {
    __threadfence_system();
    ticket = atomicAdd(sync.counter, 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0 && ticket == gridDim.x - 1) {
    *sync.counter = 0;  // reset for the next exchange (stream-ordered)
    signal_peers(sync);
  }
}

__global__ void __launch_bounds__(256)
    exchange_sp_to_tp_kernel(const float* __restrict__ src, PeerPtrs dst, int B, int T, int S,
                             int C, int t_lo, int Tl, int s_chunk, ExchangeSync sync) {
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
  finish_cta(sync);
}

__global__ void __launch_bounds__(256)
    exchange_tp_to_sp_kernel(const float* __restrict__ src, PeerPtrs dst, int B, int T, int S,
                             int C, int s_lo, int Sl, int t_chunk, ExchangeSync sync) {
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
  finish_cta(sync);
}

static int grid_for(int rows) {
  int grid = (rows + 7) / 8;
  if (grid > 4 * 148) grid = 4 * 148;
  return grid < 1 ? 1 : grid;
}

int exchange_sp_to_tp(const float* src, const PeerPtrs& dst, int B, int T, int S, int C, int P,
                      int t_lo, int Tl, const ExchangeSync& sync, cudaStream_t s) {
  const int rows = B * Tl * S;
  if (rows <= 0 && sync.flags.p[0] == nullptr) return 0;
  const int s_chunk = (S + P - 1) / P;
  exchange_sp_to_tp_kernel<<<grid_for(rows), 256, 0, s>>>(src, dst, B, T, S, C, t_lo, Tl, s_chunk,
                                                          sync);
  return 1;
}

int exchange_tp_to_sp(const float* src, const PeerPtrs& dst, int B, int T, int S, int C, int P,
                      int s_lo, int Sl, const ExchangeSync& sync, cudaStream_t s) {
  const int rows = B * T * Sl;
  if (rows <= 0 && sync.flags.p[0] == nullptr) return 0;
  const int t_chunk = (T + P - 1) / P;
  exchange_tp_to_sp_kernel<<<grid_for(rows), 256, 0, s>>>(src, dst, B, T, S, C, s_lo, Sl, t_chunk,
                                                          sync);
  return 1;
}

// Wait until every rank q published this rank's current epoch into slot q. The spin is bounded
// (globaltimer): a peer that never signals (dead process, wedged GPU) sets *status to
// DDIT_XCH_TIMEOUT and the kernel returns, so the stream drains and the host reads the error
// (ddit_request_status) instead of the GPU hanging.
__global__ void flag_wait_kernel(const uint32_t* flags, const uint32_t* epoch_p, int P,
                                 uint32_t* status, unsigned long long timeout_ns) {
  const int q = threadIdx.x;
  if (q >= P) return;
  const uint32_t epoch = *epoch_p;
  const uint32_t* mine = flags + q;
  uint32_t v;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int spin = 0;; ++spin) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
    if ((int32_t)(v - epoch) >= 0) return;
    if ((spin & 1023) == 1023) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        if (status) atomicMax(status, 1u + (uint32_t)q);  // 1 + the rank that never signalled
        return;
      }
    }
  }
}

static unsigned long long flag_timeout_ns() {
  static unsigned long long ns = 0;
  if (ns == 0) {
    const char* e = getenv("DDIT_XCH_TIMEOUT_MS");
    const double ms = e ? atof(e) : 20000.0;
    ns = (unsigned long long)((ms > 0 ? ms : 20000.0) * 1e6);
  }
  return ns;
}

int flag_wait(const uint32_t* own_flags, const uint32_t* epoch, int P, uint32_t* status,
              cudaStream_t s) {
  flag_wait_kernel<<<1, 32, 0, s>>>(own_flags, epoch, P, status, flag_timeout_ns());
  return 1;
}

}  // namespace ddit
