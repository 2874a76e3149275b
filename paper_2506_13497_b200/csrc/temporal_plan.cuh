// Host-side plan of the tcgen05 temporal-attention kernel (attention_temporal.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "ddit.h"

namespace ddit {
struct alignas(64) TemporalParams {
  CUtensorMap tmO;           // o as {72, heads, T, positions, batches}, box {72, 1, R, 1, 1}
  const __nv_bfloat16* qkv;  // row r: [q (C) | k (C) | v (C)], head h at 72 h within each
  int ld;                    // QKV row stride (elements)
  long long tok_ld;          // frame stride (elements): tok rows
  int outer;                 // batch stride (rows); positions are consecutive rows
  int T;              // frames per sequence (<= 64)
  int heads;
  int groups;         // head groups of 128 / R heads
  int inner;          // positions per batch
  int batches;        // num_seqs / inner
  float scale_log2;
};

struct TemporalPlan {
  TemporalParams p;
  int R;                      // rows per head in a tile: 16 (T <= 16), 32 (T <= 32) or 64
  dim3 grid;
};

int temporal_plan_init(TemporalPlan* tp, const ddit_attn* a);
int temporal_plan_launch(const TemporalPlan* tp, cudaStream_t s);
int temporal_attention_launch(const ddit_attn* a, cudaStream_t s);
}  // namespace ddit
