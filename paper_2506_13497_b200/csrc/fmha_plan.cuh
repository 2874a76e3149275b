// Host-side plan of the tcgen05 flash-attention kernel (fmha_sm100.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "ddit.h"

namespace ddit {
struct FmhaParams {
  int Lq, Lk;
  int q_slot, k_slot, v_slot, o_slot;  // head-slot offsets of head 0 in the maps
  float scale_log2;
  int q_tiles, heads, seqs;
};

struct FmhaPlan {
  CUtensorMap tmQa, tmQb, tmKVa, tmKVb, tmO;
  FmhaParams p;
  dim3 grid;
};

bool fmha_supported(const ddit_attn* a);
int fmha_plan_init(FmhaPlan* fp, const ddit_attn* a);
int fmha_plan_launch(const FmhaPlan* fp, cudaStream_t s);
}  // namespace ddit
