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

#include <algorithm>
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

// ---- staged all-to-all (the NCCL arm): rows packed per destination rank into one contiguous
// send buffer, exchanged by ncclAllToAll(v) on the caller's side, unpacked per source rank.
// Block order of the send buffer: destination q = 0..P-1; inside a block the rows keep the order
// of the source layout. Row = C fp32. XchGeom describes both layouts of a DoP-P group.
DDIT_DEV int chunk_lo(int X, int P, int q) { return min(q * ((X + P - 1) / P), X); }
DDIT_DEV int chunk_len(int X, int P, int q) {
  return chunk_lo(X, P, q + 1) - chunk_lo(X, P, q);
}

// dir 0 (after a spatial block): x_sp [B][Tl][S] -> blocks q of rows (b, tl, s in S_q)
// dir 1 (after a temporal block): x_tp [B][T][Sl] -> blocks q of rows (b, t in T_q, sl)
// Maps packed row i of this rank to its row in the source layout.
DDIT_DEV size_t pack_src_row(const XchGeom& g, int dir, int i) {
  int q = 0, base = 0;
  for (; q < g.P; ++q) {
    const int n = dir == 0 ? g.B * g.Tl * chunk_len(g.S, g.P, q) : g.B * chunk_len(g.T, g.P, q) * g.Sl;
    if (i < base + n) break;
    base += n;
  }
  const int j = i - base;
  if (dir == 0) {
    const int Sq = chunk_len(g.S, g.P, q), s_lo = chunk_lo(g.S, g.P, q);
    const int s = j % Sq, tl = (j / Sq) % g.Tl, b = j / (Sq * g.Tl);
    return ((size_t)b * g.Tl + tl) * g.S + s_lo + s;
  }
  const int Tq = chunk_len(g.T, g.P, q), t_lo = chunk_lo(g.T, g.P, q);
  const int sl = j % g.Sl, t = (j / g.Sl) % Tq, b = j / (g.Sl * Tq);
  return ((size_t)b * g.T + t_lo + t) * g.Sl + sl;
}
// Maps received row i (blocks from source r = 0..P-1) to its row in this rank's destination
// layout: dir 0 -> x_tp [B][T][Sl] (source r sent frames T_r), dir 1 -> x_sp [B][Tl][S].
DDIT_DEV size_t unpack_dst_row(const XchGeom& g, int dir, int i) {
  int r = 0, base = 0;
  for (; r < g.P; ++r) {
    const int n = dir == 0 ? g.B * chunk_len(g.T, g.P, r) * g.Sl : g.B * g.Tl * chunk_len(g.S, g.P, r);
    if (i < base + n) break;
    base += n;
  }
  const int j = i - base;
  if (dir == 0) {
    const int Tr = chunk_len(g.T, g.P, r), t_lo = chunk_lo(g.T, g.P, r);
    const int sl = j % g.Sl, tr = (j / g.Sl) % Tr, b = j / (g.Sl * Tr);
    return ((size_t)b * g.T + t_lo + tr) * g.Sl + sl;
  }
  const int Sr = chunk_len(g.S, g.P, r), s_lo = chunk_lo(g.S, g.P, r);
  const int s = j % Sr, tl = (j / Sr) % g.Tl, b = j / (Sr * g.Tl);
  return ((size_t)b * g.Tl + tl) * g.S + s_lo + s;
}

__global__ void __launch_bounds__(256)
    xch_pack_kernel(const float* __restrict__ src, float* __restrict__ send, XchGeom g, int dir,
                    int rows) {
  const int nv = g.C >> 2;
  for (int i = blockIdx.x * 8 + (threadIdx.x >> 5); i < rows; i += gridDim.x * 8) {
    const float4* sp = reinterpret_cast<const float4*>(src + pack_src_row(g, dir, i) * g.C);
    float4* dp = reinterpret_cast<float4*>(send + (size_t)i * g.C);
    for (int v = threadIdx.x & 31; v < nv; v += 32) dp[v] = __ldg(sp + v);
  }
}

__global__ void __launch_bounds__(256)
    xch_unpack_kernel(const float* __restrict__ recv, float* __restrict__ dst, XchGeom g, int dir,
                      int rows) {
  const int nv = g.C >> 2;
  for (int i = blockIdx.x * 8 + (threadIdx.x >> 5); i < rows; i += gridDim.x * 8) {
    const float4* sp = reinterpret_cast<const float4*>(recv + (size_t)i * g.C);
    float4* dp = reinterpret_cast<float4*>(dst + unpack_dst_row(g, dir, i) * g.C);
    for (int v = threadIdx.x & 31; v < nv; v += 32) dp[v] = __ldg(sp + v);
  }
}

void xch_counts(const XchGeom& g, int dir, int* send_rows, int* recv_rows) {
  auto lo = [](int X, int P, int q) { return std::min(q * ((X + P - 1) / P), X); };
  auto len = [&](int X, int P, int q) { return lo(X, P, q + 1) - lo(X, P, q); };
  for (int q = 0; q < g.P; ++q) {
    if (dir == 0) {
      send_rows[q] = g.B * g.Tl * len(g.S, g.P, q);
      recv_rows[q] = g.B * len(g.T, g.P, q) * g.Sl;
    } else {
      send_rows[q] = g.B * len(g.T, g.P, q) * g.Sl;
      recv_rows[q] = g.B * g.Tl * len(g.S, g.P, q);
    }
  }
}

int xch_pack(const float* src, float* send, const XchGeom& g, int dir, int rows, cudaStream_t s) {
  if (rows <= 0) return 0;
  xch_pack_kernel<<<grid_for(rows), 256, 0, s>>>(src, send, g, dir, rows);
  return 1;
}

int xch_unpack(const float* recv, float* dst, const XchGeom& g, int dir, int rows, cudaStream_t s) {
  if (rows <= 0) return 0;
  xch_unpack_kernel<<<grid_for(rows), 256, 0, s>>>(recv, dst, g, dir, rows);
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

static unsigned long long g_timeout_ns = 0;
static unsigned long long flag_timeout_ns() {
  if (g_timeout_ns == 0) {
    const char* e = getenv("DDIT_XCH_TIMEOUT_MS");
    const double ms = e ? atof(e) : 20000.0;
    g_timeout_ns = (unsigned long long)((ms > 0 ? ms : 20000.0) * 1e6);
  }
  return g_timeout_ns;
}
void set_flag_timeout_ms(double ms) { g_timeout_ns = ms > 0 ? (unsigned long long)(ms * 1e6) : 0; }

int flag_wait(const uint32_t* own_flags, const uint32_t* epoch, int P, uint32_t* status,
              cudaStream_t s) {
  flag_wait_kernel<<<1, 32, 0, s>>>(own_flags, epoch, P, status, flag_timeout_ns());
  return 1;
}

}  // namespace ddit
