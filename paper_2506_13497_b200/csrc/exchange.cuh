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
// Completion signalling of one exchange: flags.p[q] = rank q's flag array (uint32 [P]),
// counter = this rank's CTA ticket counter (device, zero-initialised).
// The epoch lives in device memory (incremented by the last CTA of every exchange), so a
// captured CUDA graph of the step stays correct on every replay.
struct ExchangeSync {
  PeerFlags flags;  // p[0] == nullptr: no signalling (virtual ranks, stream-ordered)
  unsigned int* counter;
  uint32_t* epoch;  // this rank's exchange counter
  int rank, P;
};
// Return the number of kernels launched (0 or 1).
int exchange_sp_to_tp(const float* src, const PeerPtrs& dst, int B, int T, int S, int C, int P,
                      int t_lo, int Tl, const ExchangeSync& sync, cudaStream_t s);
int exchange_tp_to_sp(const float* src, const PeerPtrs& dst, int B, int T, int S, int C, int P,
                      int s_lo, int Sl, const ExchangeSync& sync, cudaStream_t s);
// Staged all-to-all (NCCL arm): geometry of both layouts of this rank; dir 0 = after a spatial
// block (x_sp -> x_tp), 1 = after a temporal block (x_tp -> x_sp).
struct XchGeom {
  int B, T, S, C, P;
  int Tl, Sl;  // this rank's frame / token counts
};
void xch_counts(const XchGeom& g, int dir, int* send_rows, int* recv_rows);
int xch_pack(const float* src, float* send, const XchGeom& g, int dir, int rows, cudaStream_t s);
int xch_unpack(const float* recv, float* dst, const XchGeom& g, int dir, int rows, cudaStream_t s);
// Bounded wait (DDIT_XCH_TIMEOUT_MS, default 20 s): on timeout *status = 1 + the silent rank.
void set_flag_timeout_ms(double ms);  // <= 0: back to DDIT_XCH_TIMEOUT_MS / 20 s
int flag_wait(const uint32_t* own_flags, const uint32_t* epoch, int P, uint32_t* status,
              cudaStream_t s);
}  // namespace ddit
