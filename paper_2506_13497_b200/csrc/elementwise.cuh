// Declarations of the memory-bound step kernels (elementwise.cu). All return 0 or -2.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stddef.h>

namespace ddit {
void set_ln_variant(int v);
int ln_modulate(const float* x, __nv_bfloat16* out, int M, int C, const float* shift,
                const float* scale, int mod_stride, int rows_per_b, float eps, cudaStream_t s);
int timestep_freq(float* freq, const float* tvals, int nvals, int dim, cudaStream_t s);
int gemv(const __nv_bfloat16* W, const float* bias, const float* x, float* y, int nb, int N, int K,
         int in_act, int out_act, int accumulate, cudaStream_t s);
int modulation(float* mods, const float* const* sst, const float* t_mlp, int nblocks, int nb,
               int C, float* fin, const float* fsst, const float* t, cudaStream_t s);
int build_tables(float* pos, int h, int w, int C, float scale, float base_size, float* rope, int T,
                 int D, cudaStream_t s);
int patch_embed(const float* z, const float* Wp, const float* bp, const float* pos, float* x, int Tl,
                int Hl, int Wl, int h, int w, int C, int Cin, int nb, cudaStream_t s);
int final_layer(const float* x, const float* fin, const float* Wf, const float* bf, float* z, int Tl,
                int Hl, int Wl, int h, int w, int C, int Cin, int out_ch, float guidance, float dt,
                float eps, cudaStream_t s);
int cast_bf16(const float* in, __nv_bfloat16* out, size_t n, cudaStream_t s);
}  // namespace ddit
