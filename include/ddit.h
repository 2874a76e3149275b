/*
 * ddit.h -- C ABI of the B200-native DDiT hot path (libddit.so, sm_100a).
 *
 * The reference (arxiv 2506.13497, `ditsim`) has no FFI: the hot path is the Python
 * duck-typed execution model `ProfileTable.dit_step(resolution, dop) -> seconds`
 * (reference pkg/src/ditsim/profiles.py:69-76, called from engine.py:245,289,292) and
 * `ProfileTable.vae(resolution, dop)` (profiles.py:78-85, engine.py:305). This header is the
 * native boundary that replaces those lookups with real work on B200s: every entry point takes
 * plain device pointers, sizes and a cudaStream_t (passed as void*), returns 0 on success or a
 * negative DDIT_E* code, and never throws. `ddit_last_error()` gives the message of the last
 * failure on the calling thread. Only the controller thread of a process calls in.
 *
 * Python binds it with ctypes (paper_2506_13497_b200/_lib.py); INTEGRATION.md shows the
 * binding a ditsim maintainer would add.
 */
#ifndef DDIT_H_
#define DDIT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DDIT_API __attribute__((visibility("default")))

/* Error codes. Python maps DDIT_E_LOOKUP -> ProfileLookupError (profiles.py:36-37),
 * DDIT_E_ALLOC -> AllocationError (allocator.py:22-23), DDIT_E_CONFIG -> SimulationError
 * (engine.py:33-34); the others raise RuntimeError. */
#define DDIT_OK 0
#define DDIT_E_INVALID (-2)  /* bad argument / shape */
#define DDIT_E_TMA (-3)      /* tensor-map creation failed */
#define DDIT_E_CUDA (-4)     /* CUDA runtime error */
#define DDIT_E_LOOKUP (-5)   /* unknown resolution / DoP */
#define DDIT_E_ALLOC (-6)    /* device memory / group misuse */
#define DDIT_E_CONFIG (-7)   /* inconsistent configuration */

DDIT_API const char* ddit_last_error(void);
DDIT_API int ddit_version(void);
DDIT_API int ddit_num_sms(void);
/* GEMM kernel selection for plans built afterwards: 1 (default) = cta_group::2 kernel
 * (256-row tiles over a CTA pair), 0 = single-CTA kernel (128-row tiles). Env DDIT_GEMM_2CTA=0. */
DDIT_API int ddit_set_gemm_2cta(int on);
/* DoP > 1: fuse the DSP exchange into every block's fc2 GEMM -- the gated-residual epilogue
 * stores each updated row straight into its owner rank's buffer of the other layout (peer
 * memory over NVLink) and the kernel's last CTA publishes the exchange flag; 0 = the separate
 * exchange kernel. Default 1 (env DDIT_FUSED_XCH=0); applies to peers registered afterwards. */
DDIT_API int ddit_set_fused_exchange(int on);
/* Gated-residual GEMMs without a bf16 copy or fused exchange: 1 (default) = the update leaves
 * through a TMA reduce-add into the fp32 residual (no residual loads), 0 = TMA load / update /
 * store. Both give bit-identical results. Env DDIT_RESID_RED=0; applies to plans built afterwards. */
DDIT_API int ddit_set_resid_reduce(int on);
/* 2-CTA GEMMs with K >= 4096 and BN 192 (fc2) as 256 x 384 tiles -- two accumulator halves, one
 * tile in TMEM -- (default 1; env DDIT_GEMM_WIDE=0); bit-identical results. Plans built afterwards. */
DDIT_API int ddit_set_gemm_wide(int on);
/* QKV GEMM on per-head padded weights (80-row head slots, 256 x 240 tiles; default 1; env
 * DDIT_QKV_PAD=0); bit-identical results. Applies to requests opened afterwards. */
DDIT_API int ddit_set_qkv_pad(int on);
/* VAE convolutions as cta_group::2 pairs of 128-pixel tiles (half the weight rows per CTA) when
 * there are enough tiles (default 1; env DDIT_CONV_2CTA=0); bit-identical results. */
DDIT_API int ddit_set_conv_2cta(int on);
/* VAE convolution pixel tiles: R rows x Wt columns chosen per layer for the fewest tiles (1,
 * default; env DDIT_CONV_TILES=0: 128-pixel rows); bit-identical results. */
DDIT_API int ddit_set_conv_tile_search(int on);
/* Programmatic dependent launch of the step kernels (default 1; env DDIT_PDL=0). */
DDIT_API int ddit_set_pdl(int on);
/* One process driving several GPUs: let `device` access `peer`'s memory (idempotent). */
DDIT_API int ddit_enable_peer_access(int device, int peer);

/* ------------------------------------------------------------------ kernel-level ops
 * Exposed for parity tests and profiling; the step below composes them. */

/* Epilogue kinds of ddit_gemm (see csrc/gemm_sm100.cuh). */
#define DDIT_EPI_BF16 0      /* out_bf16 = A.B^T + bias */
#define DDIT_EPI_GELU_BF16 1 /* out_bf16 = gelu_tanh(A.B^T + bias) */
#define DDIT_EPI_RESID 2     /* resid_f32 += gate[b] * (A.B^T + bias) (+ bf16 copy) */
#define DDIT_EPI_QKV 3       /* bias + per-head RMSNorm on q,k + optional RoPE; bf16 out */
#define DDIT_EPI_F32 4       /* out_f32 = A.B^T + bias */

typedef struct ddit_epi {
  const float* bias;   /* [N] fp32 or NULL */
  void* out;           /* bf16 [M, ldo] (DDIT_EPI_F32: fp32) */
  int ldo;
  float* resid;        /* DDIT_EPI_RESID: fp32 [M, ldr] */
  int ldr;
  const float* gate;   /* DDIT_EPI_RESID: fp32 [B][gate_stride] or NULL (gate = 1) */
  int gate_stride;
  int rows_per_b;      /* row r belongs to batch r / rows_per_b */
  void* out2;          /* DDIT_EPI_RESID: optional bf16 copy of the new residual */
  int ldo2;
  const float* qnorm_w; /* DDIT_EPI_QKV: [72] */
  const float* knorm_w; /* DDIT_EPI_QKV: [72] */
  int hidden;          /* DDIT_EPI_QKV: C (q = cols [0,C), k = [C,2C), v = [2C,3C)) */
  int rope;            /* DDIT_EPI_QKV: 1 = rotate q,k by frame index */
  int rope_T;          /* frames */
  int rope_S;          /* rows per frame in this layout: t = (row / rope_S) % rope_T */
  const float* rope_tab; /* [rope_T][36][2] (cos, sin) */
  float eps;
} ddit_epi;

/* D = A[M,K] . B[N,K]^T on tcgen05 (bf16 in, fp32 accumulate) with a fused epilogue.
 * bn in {128,144,192,256}; N % bn == 0; K % 64 == 0. */
DDIT_API int ddit_gemm(const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                       int epi, const ddit_epi* ep, int bn, void* stream);

/* Flash attention over bf16 q/k/v (head_dim 72). Token j of sequence i lives at row
 *   (i / inner) * outer + (i % inner) * inner_stride + j * tok
 * of the q (and o) matrix, and likewise with the kv_* map for k and v; head h occupies
 * columns [72h, 72h+72). Covers spatial, temporal and cross attention without re-layout. */
typedef struct ddit_attn {
  const void* q; int ldq;
  const void* k; int ldk;
  const void* v; int ldv;
  void* o; int ldo;
  int heads;
  int head_dim;
  int num_seqs;
  int Lq, Lk;
  int q_inner, q_outer, q_inner_stride, q_tok;
  int kv_inner, kv_outer, kv_inner_stride, kv_tok;
  float scale;
} ddit_attn;

/* Temporal attention (T <= 64 frames; tcgen05): q/k/v must be the three sections of one
 * row-major QKV matrix and share one index map (heads of one position stacked into 128-row tiles). */
DDIT_API int ddit_attention_temporal(const ddit_attn* a, void* stream);
/* LayerNorm (no affine, eps) + t2i modulate of the fp32 residual rows:
 * out_bf16[r, :] = LN(x[r, :]) * (1 + scale[b]) + shift[b], b = r / rows_per_b, shift / scale
 * rows mod_stride floats apart. The step's own LN launch (same kernel). */
DDIT_API int ddit_ln_modulate(const float* x, void* out_bf16, int M, int C, const float* shift,
                              const float* scale, int mod_stride, int rows_per_b, float eps,
                              void* stream);
/* LN kernel variant for launches made afterwards (tuning): 1 one warp per row, 3 persistent
 * streaming warps, 5 (default) streaming warps with the modulation held in registers (C = 1152;
 * other widths take the generic kernel); all bit-identical. Env DDIT_LN. */
DDIT_API int ddit_set_ln_variant(int variant);
/* tcgen05 / TMEM flash attention (spatial and cross attention): contiguous sequences
 * (tok == 1, inner <= 1), row strides and head offsets in whole 72-column slots, k and v in one
 * matrix. Returns DDIT_E_INVALID for layouts it does not cover. */
DDIT_API int ddit_attention_tc(const ddit_attn* a, void* stream);

/* ------------------------------------------------------------------ the STDiT3 step
 * Model = device weights (caller-owned, registered by pointer). Request = one video being
 * denoised on one rank of a DoP-P group: shard geometry, workspace (caller-allocated), cached
 * text embedding and per-block cross-attention K/V. The step replaces the reference's
 * `ProfileTable.dit_step(res, dop)` lookup (profiles.py:69-76) at the engine's step sites
 * (engine.py:245 start, :289 after a promotion, :292 steady state). */

typedef struct ddit_config {
  int depth;            /* 28 (spatial + temporal block pairs) */
  int hidden;           /* C = 1152 */
  int heads;            /* 16 */
  int head_dim;         /* 72 */
  int mlp_hidden;       /* 4608 */
  int in_channels;      /* 4 */
  int out_channels;     /* 8 (pred_sigma) */
  int caption_channels; /* 4096 */
  int text_tokens;      /* 300 */
  int freq_dim;         /* 256 */
  int input_sq_size;    /* 512 */
  float eps;            /* 1e-6 */
} ddit_config;

/* Linear weights are bf16 [out, in] (nn.Linear layout); biases, tables and norms fp32. */
typedef struct ddit_block_weights {
  const float* scale_shift_table; /* [6, C] */
  const void* qkv_w; const float* qkv_b;
  const float* q_norm; const float* k_norm;
  const void* proj_w; const float* proj_b;
  const void* cq_w; const float* cq_b;
  const void* ckv_w; const float* ckv_b;
  const void* cproj_w; const float* cproj_b;
  const void* fc1_w; const float* fc1_b;
  const void* fc2_w; const float* fc2_b;
} ddit_block_weights;

typedef struct ddit_weights {
  const float* x_emb_w;  /* fp32 [C, in*4] (Conv3d (1,2,2) flattened) */
  const float* x_emb_b;
  const void* t0_w; const float* t0_b; /* t_embedder.mlp.0: bf16 [C, 256] */
  const void* t2_w; const float* t2_b; /* t_embedder.mlp.2: bf16 [C, C] */
  const void* f0_w; const float* f0_b; /* fps_embedder.mlp.0 */
  const void* f2_w; const float* f2_b; /* fps_embedder.mlp.2 */
  const void* tb_w; const float* tb_b; /* t_block.1: bf16 [6C, C] */
  const void* y1_w; const float* y1_b; /* y_embedder fc1: bf16 [C, 4096] */
  const void* y2_w; const float* y2_b; /* y_embedder fc2: bf16 [C, C] */
  const float* y_null;                 /* fp32 [300, 4096] */
  const float* final_sst;              /* fp32 [2, C] */
  const float* final_w;                /* fp32 [out*4, C] */
  const float* final_b;                /* fp32 [out*4] */
  const ddit_block_weights* blocks;    /* host array of 2*depth: spatial i at 2i, temporal 2i+1 */
} ddit_weights;

typedef struct ddit_req_desc {
  int latent_t, latent_h, latent_w; /* z is [1, 4, T, Hl, Wl] */
  int height, width;                /* pixels: pos-embed scale and timestep transform */
  int dop, rank;                    /* DoP P in {1,2,4,8}; this rank */
  int num_steps;                    /* 30 */
  float guidance;                   /* 7.0 */
  float fps;                        /* 24 */
} ddit_req_desc;

typedef struct ddit_model ddit_model;
typedef struct ddit_req ddit_req;

DDIT_API int ddit_model_create(const ddit_config* cfg, const ddit_weights* w, ddit_model** out);
DDIT_API void ddit_model_destroy(ddit_model* m);

/* Bytes of device workspace a request needs (caller allocates, 256-byte aligned). */
DDIT_API int ddit_request_workspace_bytes(const ddit_model* m, const ddit_req_desc* d,
                                          uint64_t* bytes);
/* Shard of this rank: frames [t_lo, t_hi) (spatial phase) and tokens [s_lo, s_hi) (temporal).
 * Pure host arithmetic (m may be NULL): rank r owns [r*ceil(X/P), (r+1)*ceil(X/P)) ∩ [0, X). */
DDIT_API int ddit_request_shard(const ddit_model* m, const ddit_req_desc* d, int* t_lo, int* t_hi,
                                int* s_lo, int* s_hi);
/* Opens a request: builds tables, embeds the caption y_cond (device fp32 [300, 4096]) together
 * with the null caption, caches the per-block cross-attention K/V. */
DDIT_API int ddit_request_open(ddit_model* m, const ddit_req_desc* d, void* workspace,
                               uint64_t bytes, const float* y_cond, void* stream, ddit_req** out);
DDIT_API void ddit_request_close(ddit_req* r);
/* Re-bind an open request (same shape / DoP / rank) to a new caption: recomputes the text
 * embedding and the cross-attention K/V cache. Lets a serving loop keep pools of opened rank
 * states (workspace, tables, GEMM / attention plans) instead of re-opening per request. */
DDIT_API int ddit_request_set_text(ddit_req* r, const float* y_cond, void* stream);
/* Promotion / re-shard broadcast (reference OverheadModel.broadcast_seconds, engine.py:52-61):
 * copy src's text embedding and cross-attention K/V cache into dst (same model; dst may live on
 * another peer-enabled device -- the copy then crosses NVLink). */
DDIT_API int ddit_request_copy_text(ddit_req* dst, const ddit_req* src, void* stream);
/* Cheaper promotion broadcast: copy only src's y-embedding (B*300 x C bf16) into dst and
 * recompute the 2*depth cross-attention K/V projections on dst's device (same result bit for bit
 * as ddit_request_copy_text; per new rank 1.4 MB over NVLink + 56 small GEMMs instead of 155 MB). */
DDIT_API int ddit_request_share_text(ddit_req* dst, const ddit_req* src, void* stream);
/* Promotion P -> P' for a whole new group in one call (SURVEY §8(b) ddit_reshard): rank i of the
 * new group (new_ranks[i], its z shard new_z[i], on its own device / streams[i] or the legacy
 * stream when streams is NULL) gathers its frames [t_lo, t_hi) from the p old shards old_z[k]
 * (frames [old_t_lo[k], old_t_hi[k]), peer pointers) and takes its text state from text_src
 * (ddit_request_share_text). Replaces OverheadModel.broadcast_seconds + scale_up_seconds
 * (reference engine.py:52-61, applied at :281-290). */
DDIT_API int ddit_reshard(ddit_req* const* new_ranks, float* const* new_z, int q,
                          const float* const* old_z, const int* old_t_lo, const int* old_t_hi,
                          int p, const ddit_req* text_src, void* const* streams);
/* Device ms of the last ddit_reshard work into rank r (synchronises on it). */
DDIT_API int ddit_request_reshard_ms(ddit_req* r, float* ms);

/* DoP > 1: register every rank's exchange buffers (x_sp, x_tp: fp32, as returned by
 * ddit_request_exchange_buffers on that rank, peer-mapped) and flag arrays (uint32 [P]). */
DDIT_API int ddit_request_exchange_buffers(ddit_req* r, void** x_sp, void** x_tp, void** flags);
DDIT_API int ddit_request_set_peers(ddit_req* r, void* const* x_sp, void* const* x_tp,
                                    void* const* flags);

/* One full denoise step on this rank. z_local: device fp32 [4][t_hi-t_lo][Hl][Wl], updated
 * in place (z <- z + v * dt). For DoP > 1 every rank of the group calls it concurrently. */
DDIT_API int ddit_dit_step(ddit_req* r, float* z_local, int step, void* stream);

/* The same step split into phases (virtual ranks on one device drive these in lockstep):
 * begin (t-embedding, modulation table, patch embed), phase k in [0, 2*depth) = block k
 * followed by the push half of the exchange, end (final layer, CFG, Euler). */
DDIT_API int ddit_step_begin(ddit_req* r, const float* z_local, int step, void* stream);
DDIT_API int ddit_step_phase(ddit_req* r, int phase, void* stream);
DDIT_API int ddit_step_end(ddit_req* r, float* z_local, int step, void* stream);
/* Cross-rank barrier after a push (no-op at DoP 1). */
DDIT_API int ddit_step_barrier(ddit_req* r, void* stream);
/* Health of a DoP > 1 request after its stream ran (synchronises `stream`): the barrier spin is
 * bounded (env DDIT_XCH_TIMEOUT_MS, default 20000); status = 0 ok, or 1 + the rank whose flag
 * never arrived, returned with DDIT_E_CONFIG. */
DDIT_API int ddit_request_status(ddit_req* r, void* stream, uint32_t* status);
/* Bound of the barrier spin in ms for launches from now on (<= 0: DDIT_XCH_TIMEOUT_MS / 20 s). */
DDIT_API int ddit_set_exchange_timeout_ms(int ms);

/* Device timestep (after the RFLOW transform) and dt of a step, for logging / tests. */
DDIT_API int ddit_request_timestep(const ddit_req* r, int step, float* t, float* dt);

/* Request options: DDIT_OPT_TC_ATTENTION is retired -- spatial / cross attention always run the
 * tcgen05 FMHA (value 1 is accepted, 0 returns DDIT_E_INVALID; there is no other attention
 * kernel). */
#define DDIT_OPT_TC_ATTENTION 1
/* DDIT_OPT_EXTERNAL_XCH (default 0): the step does not exchange rows itself (no peers, no fused
 * fc2 stores, no flag barrier); after every ddit_step_phase the caller moves them with
 * ddit_request_xch_pack -> an all-to-all (ncclAllToAll in dist.NcclGroupStep) ->
 * ddit_request_xch_unpack. The baseline the fused peer-store exchange is measured against. */
#define DDIT_OPT_EXTERNAL_XCH 2
DDIT_API int ddit_request_set_option(ddit_req* r, int option, int value);

/* Profiling: while enabled every launch of the request is bracketed by CUDA events on its
 * stream; _read returns per-class totals (ms, launches) for classes
 * 0 = tcgen05 GEMM, 1 = attention, 2 = elementwise / embed / final, 3 = exchange + barrier,
 * and resets. */
/* Staged all-to-all after phase `phase` (even: spatial block, x_sp -> x_tp; odd: temporal,
 * x_tp -> x_sp). Rows are C fp32. xch_counts: rows this rank sends to / receives from every
 * rank q (arrays of dop ints). xch_pack writes the rows into `send` grouped by destination rank
 * (contiguous, rank order); xch_unpack scatters `recv` (grouped by source rank) into the other
 * layout. Replaces the paper's NCCL all-to-all between sequence-parallel workers
 * (reference engine.py:286-290 only charges a constant). */
DDIT_API int ddit_request_xch_counts(ddit_req* r, int phase, int* send_rows, int* recv_rows);
DDIT_API int ddit_request_xch_pack(ddit_req* r, int phase, void* send, void* stream);
DDIT_API int ddit_request_xch_unpack(ddit_req* r, int phase, const void* recv, void* stream);
DDIT_API int ddit_request_profile(ddit_req* r, int enable);
DDIT_API int ddit_request_profile_read(ddit_req* r, float* ms, int* count);
/* Total kernel launches issued by libddit in this process. */
DDIT_API unsigned long long ddit_launch_count(void);

/* ------------------------------------------------------------------ VAE decode kernels (K13)
 * Implicit-GEMM convolution on tcgen05 over channels-last bf16 activations [B][T][H][W][C]
 * (T = 1 for 2-D). Weights bf16 [Cout][kt][kh][kw][Cin]; "same" zero padding in H, W; in T
 * either centred or causal (kt-1 frames of zeros in front, OpenSora CausalConv3d). Optional
 * fp32 bias [Cout] and bf16 residual [B][T][H][W][Cout] added in the epilogue.
 * Cin, Cout multiples of 64. */
typedef struct ddit_conv_args {
  const void* x;
  void* y;
  const void* w;
  const float* bias;
  const void* residual;
  int B, T, H, W, Cin, Cout;
  int kt, kh, kw;
  int causal_time;
  /* optional (NULL = off): GroupNorm statistics of y for gn_groups groups, written by the
   * epilogue as fp32 (sum, sum of squares) pairs over the in-frame pixels of each pixel tile:
   * per frame [B*T][gn_groups][nblk], nblk = ddit_conv_frame_tiles(H, W), or with gn_per_sample
   * per sample [B][gn_groups][T*nblk]; the input of ddit_groupnorm_partials. Needs
   * Cout / gn_groups in {2, 4, 8, 16, 32, 64}. */
  float* gn_part;
  int gn_groups;
  int gn_per_sample;
} ddit_conv_args;
DDIT_API int ddit_conv(const ddit_conv_args* a, void* stream);
/* pixel tiles per H x W frame of ddit_conv (the nblk of its GroupNorm partials) */
DDIT_API int ddit_conv_frame_tiles(int H, int W);

/* GroupNorm over channels-last x [N][P][C] bf16 (per sample n, group of C/G channels, all P
 * pixels), affine, optional SiLU -> y bf16. Deterministic (fixed reduction order).
 * stats: device scratch of at least N*G*2 doubles + N*512*G float2 (partials) + N*C float2
 * (per-channel affine coefficients). */
DDIT_API int ddit_groupnorm(const void* x, void* y, double* stats, const float* gamma,
                            const float* beta, int N, int P, int C, int G, float eps, int silu_act,
                            void* stream);
/* The same GroupNorm from statistics partials [N][G][nblk] (sum, sum of squares) that the
 * producing ddit_conv wrote (gn_part): no statistics pass over x. coef: device scratch of N*C
 * float2. */
DDIT_API int ddit_groupnorm_partials(const void* x, void* y, const float* partial, int nblk,
                                     float* coef, const float* gamma, const float* beta, int N,
                                     int P, int C, int G, float eps, int silu_act, void* stream);
/* nearest 2x in H and W: [N][H][W][C] -> [N][2H][2W][C] bf16 */
DDIT_API int ddit_upsample2x(const void* x, void* y, int N, int H, int W, int C, void* stream);
/* OpenSora temporal upsampling: [B][T][HW][2C] (channel 2c+ts) -> [B][2T][HW][C] bf16 */
DDIT_API int ddit_depth_to_time(const void* x, void* y, int B, int T, int HW, int C, void* stream);
/* Direct conv (CUDA cores) for layers with < 64 channels on one side. x strided
 * (x_strides = element strides {b, c, t, h, w}, NULL = dense channels-last), bf16 or fp32;
 * w fp32 [kt][kh][kw][Cin][Cout]; y bf16 channels-last, or fp32 [B][Cout][T][Hc][Wc] cropped
 * when out_cf. */
DDIT_API int ddit_conv_small(const void* x, int x_is_f32, const long long* x_strides,
                             const float* w, const float* bias, void* y, int B, int T, int H, int W,
                             int Cin, int Cout, int kt, int kh, int kw, int causal_time, int out_cf,
                             int Hc, int Wc, void* stream);
/* decoded frames: channels [0, C) of bf16 channels-last y [N][H][W][ld] -> fp32 [C][N][Hc][Wc]
 * (the video tensor [1][C][N][Hc][Wc], cropped to Hc x Wc) */
DDIT_API int ddit_frames_out(const void* y, float* out, int N, int H, int W, int ld, int C, int Hc,
                             int Wc, void* stream);
/* mid-block attention helpers: row softmax (fp32 S -> bf16 P, columns >= valid -> 0),
 * bf16 transpose with zero-padded output rows, y = bf16(a_f32 + b_bf16) */
DDIT_API int ddit_softmax_rows(const float* S, void* P, int rows, int cols, int valid, float scale,
                               void* stream);
DDIT_API int ddit_transpose_bf16(const void* in, void* out, int rows, int cols, int ld_in,
                                 int rows_pad, void* stream);
DDIT_API int ddit_add_f32_bf16(const float* a, const void* b, void* y, uint64_t n, void* stream);

/* ------------------------------------------------------------------ re-sharding (K11 / K12)
 * dst (fp32 [channels][t_hi-t_lo][hw], this rank's new T-shard) <- frames gathered from up to
 * 16 source shards src[k] ([channels][src_t_hi[k]-src_t_lo[k]][hw], peer or local pointers).
 * Promotion P -> P' (reference engine.py:281-290) and the DiT -> VAE hand-off to the vae_dop
 * lowest-id GPUs (policies.py:175-190) are both this gather. */
DDIT_API int ddit_latent_gather(float* dst, int t_lo, int t_hi, const float* const* src,
                                const int* src_t_lo, const int* src_t_hi, int nsrc, int channels,
                                int hw, void* stream);

/* ------------------------------------------------------------------ cross-process mapping
 * One process per GPU: a rank exports the (allocation handle, offset) of its exchange buffers
 * and the group's other ranks map them (peer access over NVLink). handle = 64 bytes. */
DDIT_API int ddit_ipc_export(const void* ptr, void* handle, uint64_t* offset);
DDIT_API int ddit_ipc_import(const void* handle, uint64_t offset, void** ptr);
DDIT_API int ddit_ipc_close(void* ptr, uint64_t offset);

#ifdef __cplusplus
}
#endif
#endif /* DDIT_H_ */
