// Sequence-parallel exchange (DSP all-to-all) and the cross-rank flag barrier.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ddit {
static constexpr int kMaxDop = 8;
struct PeerPtrs {
  float* p[kMaxDop];
};
struct PeerFlags {
  uint32_t* p[kMaxDop];
};
int exchange_sp_to_tp(const float* src, const PeerPtrs& dst, int B, int T, int S, int C, int P,
                      int t_lo, int Tl, cudaStream_t s);
int exchange_tp_to_sp(const float* src, const PeerPtrs& dst, int B, int T, int S, int C, int P,
                      int s_lo, int Sl, cudaStream_t s);
int flag_barrier(const PeerFlags& flags, int rank, int P, uint32_t epoch, cudaStream_t s);
}  // namespace ddit
