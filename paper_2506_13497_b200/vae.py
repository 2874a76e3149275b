"""B200 VAE decode: the real work behind the reference's
``ProfileTable.vae(resolution, dop)`` lookup (reference pkg/src/ditsim/profiles.py:78-85,
called at engine.py:305).

Every convolution with >= 64 channels on both sides runs as a tcgen05 implicit GEMM
(``ddit_conv``: TMA-shifted input windows, causal time padding by out-of-bounds zero fill);
GroupNorm(+SiLU), nearest upsampling and the temporal depth-to-time are memory-bound kernels;
the two layers with 4 latent channels use direct CUDA-core convs; the single-head mid-block
attention uses the tcgen05 GEMM + a row softmax. Activations are channels-last bf16
``[B][T][H][W][C]`` in device buffers (torch is only the allocator). Structure:
OpenSora ``VideoAutoencoderPipeline.decode`` = temporal VAE per 17-frame micro-batch then the
SDXL spatial decoder per frame (oracle: oracle/vae.py).
"""

from __future__ import annotations

import ctypes
import math
import os

import torch

from . import _lib
from ._lib import ConvArgs, check, lib, ptr, stream_ptr
from .kernels import gemm
from .vae_weights import VAEConfig

vp = ctypes.c_void_p


def _bf16(t):
    return t.to(torch.bfloat16).contiguous()


def _small(w: torch.Tensor) -> torch.Tensor:
    """fp32 [Cout][kt][kh][kw][Cin] -> [kt][kh][kw][Cin][Cout] (ddit_conv_small's layout)."""
    return w.float().permute(1, 2, 3, 4, 0).contiguous()


class VAEDecoder:
    """OpenSora-1.2 VAE decoder with device-resident weights on one GPU."""

    def __init__(self, cfg: VAEConfig, weights: dict[str, torch.Tensor], device="cuda:0",
                 graphs: int = 0, gn_from_conv: bool | None = None):
        """``graphs``: how many decode shapes keep a captured CUDA graph (0 = always eager). Off
        by default: a graph's private pool keeps every activation of the decode resident (720p:
        ~150 GB) for ~3 % at 240p, where the kernels already hide the launch overhead.
        ``gn_from_conv``: GroupNorms of a convolution's output (per frame in the spatial decoder,
        per clip in the temporal VAE) take their statistics from that convolution's epilogue (per
        pixel tile, ``ddit_conv`` gn_part) instead of a statistics pass over the activation
        (``ddit_groupnorm``); default on (env
        DDIT_VAE_GN_CONV=0: off)."""
        self.cfg = cfg
        if gn_from_conv is None:
            gn_from_conv = os.environ.get("DDIT_VAE_GN_CONV", "1") != "0"
        self.gn_from_conv = gn_from_conv
        self._gn_src = None  # (conv output tensor, its statistics partials, nblk)
        self._gn_bufs: list[torch.Tensor] = []  # partial buffers (kept alive: graphs hold them)
        self.gn_coef = torch.empty(256 * 2048 * 2, dtype=torch.float32, device=device)
        self.max_graphs = graphs
        self._graphs: dict = {}
        self.dev = torch.device(device)
        d = self.dev
        W = {k: v.to(d) for k, v in weights.items()}
        self.W = W
        # fold z * scale + shift into the temporal post_quant_conv (1x1x1: exact)
        sc = torch.tensor(cfg.scale, device=d)
        sh = torch.tensor(cfg.shift, device=d)
        wq = W["t.post_quant_conv.weight"]  # [4, 1, 1, 1, 4]
        self.t_pq_w = _small(wq * sc.view(1, 1, 1, 1, -1))
        self.t_pq_b = (W["t.post_quant_conv.bias"] + (wq[:, 0, 0, 0, :] * sh).sum(-1)).contiguous()
        # fold 1 / scaling_factor into the spatial post_quant_conv (1x1: exact)
        self.s_pq_w = _small(W["s.post_quant_conv.weight"] / cfg.scaling_factor)
        # direct (CUDA-core) convs take fp32 weights [kt][kh][kw][Cin][Cout]
        self.small = {k: _small(W[k]) for k in ("t.conv1.weight", "s.conv_in.weight")}
        self.s_pq_b = W["s.post_quant_conv.bias"].contiguous()
        self.bf: dict[str, torch.Tensor] = {}
        for k, v in list(W.items()):
            if k.endswith(".weight") and v.dim() == 5:
                cout, cin = v.shape[0], v.shape[-1]
                if cin % 64 == 0 and cout % 64 == 0:
                    self.bf[k] = _bf16(v)
                elif cin % 64 == 0:  # few output channels (conv_out): pad Cout to 64 with zeros
                    pad = torch.zeros((64, *v.shape[1:]), device=d)
                    pad[:cout] = v
                    self.bf[k] = _bf16(pad)
                    b = W.get(k[:-7] + ".bias")
                    if b is not None:
                        bp = torch.zeros(64, device=d)
                        bp[:cout] = b
                        W[k[:-7] + ".bias_pad"] = bp
        a = "s.mid.attn."
        self.w_qkv = _bf16(torch.cat([W[a + "to_q.weight"], W[a + "to_k.weight"], W[a + "to_v.weight"]]))
        self.b_qkv = torch.cat([W[a + "to_q.bias"], W[a + "to_k.bias"], W[a + "to_v.bias"]]).contiguous()
        self.w_out = _bf16(W[a + "to_out.weight"])
        # GroupNorm scratch: fp64 [N][G][2] + fp32x2 partials [N][512][G] + fp32x2 coefficients
        # [N][C], N <= 256 samples, C <= 2048
        self.stats = torch.empty(256 * 32 * 2 + 256 * 512 * 32 + 256 * 2048, dtype=torch.float64, device=d)
        self.launches = 0

    # ---------------------------------------------------------------- primitives
    def _gn_partials(self, n: int) -> torch.Tensor:
        """A partial buffer of >= n floats (a new one when the current is too small; old ones stay
        alive because captured graphs write to them)."""
        if not self._gn_bufs or self._gn_bufs[-1].numel() < n:
            self._gn_bufs.append(torch.empty(max(n, 1 << 20), dtype=torch.float32, device=self.dev))
        return self._gn_bufs[-1]

    def _conv(self, x, name, *, residual=None, bias=True, causal=True, pad_bias=False,
              gn_stats=False):
        """``gn_stats``: the epilogue also writes the GroupNorm statistics of y (per pixel tile;
        per frame for the spatial, per clip for the causal temporal convs), which the next
        ``_gn`` of exactly this tensor consumes."""
        B, T, H, Wd, Cin = x.shape
        w = self.bf[name + ".weight"]
        Cout, kt, kh, kw, _ = w.shape
        b = self.W.get(name + (".bias_pad" if pad_bias else ".bias")) if bias else None
        y = torch.empty((B, T, H, Wd, Cout), dtype=torch.bfloat16, device=self.dev)
        args = ConvArgs(ptr(x), ptr(y), ptr(w), ptr(b) if b is not None else None,
                        ptr(residual) if residual is not None else None, B, T, H, Wd, Cin, Cout, kt,
                        kh, kw, 1 if causal else 0)
        gn = None
        if gn_stats and self.gn_from_conv:
            G = self.cfg.groups
            nblk = lib().ddit_conv_frame_tiles(H, Wd) * (T if causal else 1)
            part = self._gn_partials(B * T * G * nblk * 2 // (T if causal else 1))
            args.gn_part = ptr(part)
            args.gn_groups = G
            args.gn_per_sample = 1 if causal else 0  # temporal VAE: GroupNorm over the whole clip
            gn = (y, part, nblk, not causal)
        check(lib().ddit_conv(ctypes.byref(args), stream_ptr()))
        self._gn_src = gn
        self.launches += 1
        return y

    def _conv_small(self, x, w, b, *, out_shape, causal=True, x_f32=False, strides=None,
                    out_cf=False, crop=(0, 0)):
        B, T, H, Wd, Cout = out_shape
        kt, kh, kw, Cin, Cout_w = w.shape
        if out_cf:
            y = torch.empty((B, Cout, T, crop[0], crop[1]), dtype=torch.float32, device=self.dev)
        else:
            y = torch.empty(out_shape, dtype=torch.bfloat16, device=self.dev)
        st = (ctypes.c_longlong * 5)(*strides) if strides is not None else None
        check(lib().ddit_conv_small(ptr(x), 1 if x_f32 else 0, st, ptr(w), ptr(b),
                                    ptr(y), B, T, H, Wd, Cin, Cout, kt, kh, kw, 1 if causal else 0,
                                    1 if out_cf else 0, crop[0], crop[1], stream_ptr()))
        self.launches += 1
        return y

    def _gn(self, x, name, eps, silu=True, per_frame=False):
        B, T, H, Wd, C = x.shape
        N, P = (B * T, H * Wd) if per_frame else (B, T * H * Wd)
        y = torch.empty_like(x)
        src = self._gn_src
        if src is not None and src[0] is x and src[3] == per_frame:  # statistics from the conv epilogue
            check(lib().ddit_groupnorm_partials(ptr(x), ptr(y), ptr(src[1]), src[2], ptr(self.gn_coef),
                                                ptr(self.W[name + ".weight"]), ptr(self.W[name + ".bias"]),
                                                N, P, C, self.cfg.groups, eps, 1 if silu else 0,
                                                stream_ptr()))
            self.launches += 2
            return y
        check(lib().ddit_groupnorm(ptr(x), ptr(y), ptr(self.stats), ptr(self.W[name + ".weight"]),
                                   ptr(self.W[name + ".bias"]), N, P, C, self.cfg.groups, eps,
                                   1 if silu else 0, stream_ptr()))
        self.launches += 2
        return y

    # ---------------------------------------------------------------- temporal VAE
    def _t_res(self, x, name):
        cfg = self.cfg
        h = self._gn(x, name + ".norm1", cfg.t_eps)
        h = self._conv(h, name + ".conv1", bias=False, gn_stats=True)
        h = self._gn(h, name + ".norm2", cfg.t_eps)
        res = x if (name + ".conv3.weight") not in self.W else self._conv(x, name + ".conv3", bias=False)
        return self._conv(h, name + ".conv2", residual=res, bias=False, gn_stats=True)

    def temporal_decode(self, z, t0: int, t1: int, num_frames: int) -> torch.Tensor:
        """Latent frames [t0, t1) of z [1, 4, T, h, w] (fp32, channels-first) ->
        [1, num_frames, h, w, 64] bf16 (4 valid channels)."""
        cfg = self.cfg
        _, C4, T, h, w = z.shape
        tf = cfg.time_factor
        tpad = 0 if num_frames % tf == 0 else tf - num_frames % tf
        zc = z[:, :, t0:t1]
        st = [zc.stride(0), zc.stride(1), zc.stride(2), zc.stride(3), zc.stride(4)]
        x = self._conv_small(zc, self.t_pq_w, self.t_pq_b, out_shape=(1, t1 - t0, h, w, C4),
                             x_f32=True, strides=st)
        x = self._conv_small(x, self.small["t.conv1.weight"], self.W["t.conv1.bias"],
                             out_shape=(1, t1 - t0, h, w, self.W["t.conv1.weight"].shape[0]))
        for i in range(cfg.t_res_blocks):
            x = self._t_res(x, f"t.res_blocks.{i}")
        for i in reversed(range(len(cfg.t_mults))):
            for j in range(cfg.t_res_blocks):
                x = self._t_res(x, f"t.block_res_blocks.{i}.{j}")
            if i > 0 and cfg.t_downsample[i - 1]:
                y = self._conv(x, f"t.conv_blocks.{i - 1}")
                B, Tt, H, Wd, C2 = y.shape
                x = torch.empty((B, 2 * Tt, H, Wd, C2 // 2), dtype=torch.bfloat16, device=self.dev)
                check(lib().ddit_depth_to_time(ptr(y), ptr(x), B, Tt, H * Wd, C2 // 2, stream_ptr()))
                self.launches += 1
        x = self._gn(x, "t.norm1", cfg.t_eps)
        x = self._conv(x, "t.conv_out", pad_bias=True)
        return x[:, tpad:]

    # ---------------------------------------------------------------- spatial VAE
    def _s_res(self, x, name, stats_out=True):
        """``stats_out``: a per-frame GroupNorm consumes the output (conv2 writes its statistics)."""
        cfg = self.cfg
        h = self._gn(x, name + ".norm1", cfg.sd_eps, per_frame=True)
        h = self._conv(h, name + ".conv1", causal=False, gn_stats=True)
        h = self._gn(h, name + ".norm2", cfg.sd_eps, per_frame=True)
        res = x
        if (name + ".conv_shortcut.weight") in self.W:
            res = self._conv(x, name + ".conv_shortcut", causal=False)
        return self._conv(h, name + ".conv2", residual=res, causal=False, gn_stats=stats_out)

    def _mid_attention(self, x):
        cfg = self.cfg
        N, _, H, Wd, C = x.shape  # frames as batch, T = 1
        HW = H * Wd
        HWp = -(-HW // 128) * 128
        h = self._gn(x, "s.mid.attn.group_norm", cfg.sd_eps, silu=False, per_frame=True)
        out = torch.empty_like(x)
        qkv = torch.zeros((HWp, 3 * C), dtype=torch.bfloat16, device=self.dev)
        S = torch.empty((HW, HWp), dtype=torch.float32, device=self.dev)
        P = torch.empty((HW, HWp), dtype=torch.bfloat16, device=self.dev)
        vt = torch.empty((C, HWp), dtype=torch.bfloat16, device=self.dev)
        o = torch.empty((HW, C), dtype=torch.bfloat16, device=self.dev)
        tmp = torch.empty((HW, C), dtype=torch.float32, device=self.dev)
        hf = h.view(N, HW, C)
        xf = x.view(N, HW, C)
        of = out.view(N, HW, C)
        pick = lambda n: next(b for b in (256, 192, 128, 96) if n % b == 0)  # noqa: E731
        for f in range(N):
            gemm(hf[f], self.w_qkv, bias=self.b_qkv, out=qkv[:HW], bn=pick(3 * C))
            gemm(qkv[:HW, :C], qkv[:, C:2 * C], epi=_lib.EPI_F32, out=S, bn=pick(HWp))
            check(lib().ddit_softmax_rows(ptr(S), ptr(P), HW, HWp, HW, 1.0 / math.sqrt(C), stream_ptr()))
            check(lib().ddit_transpose_bf16(ptr(qkv[:, 2 * C:]), ptr(vt), HW, C, 3 * C, HWp, stream_ptr()))
            gemm(P, vt, out=o, bn=pick(C))
            gemm(o, self.w_out, bias=self.W["s.mid.attn.to_out.bias"], epi=_lib.EPI_F32, out=tmp, bn=pick(C))
            check(lib().ddit_add_f32_bf16(ptr(tmp), ptr(xf[f]), ptr(of[f]), HW * C, stream_ptr()))
            self.launches += 7
        return out

    def spatial_decode(self, x4: torch.Tensor, height: int, width: int) -> torch.Tensor:
        """x4: [1, F, h, w, 64] bf16 (4 valid channels) -> frames fp32 [1, 3, F, height, width]."""
        cfg = self.cfg
        _, Fr, h, w, ld = x4.shape
        N = Fr
        st = [0, 1, ld * w * h, ld * w, ld]  # b, c, t(=frame), h, w
        x = self._conv_small(x4, self.s_pq_w, self.s_pq_b, out_shape=(1, N, h, w, 4), strides=st,
                             causal=False)
        x = x.view(N, 1, h, w, 4)
        top = self.W["s.conv_in.weight"].shape[0]
        x = self._conv_small(x, self.small["s.conv_in.weight"], self.W["s.conv_in.bias"],
                             out_shape=(N, 1, h, w, top), causal=False)
        x = self._s_res(x, "s.mid.resnets.0")
        x = self._mid_attention(x)
        x = self._s_res(x, "s.mid.resnets.1")
        n = len(cfg.block_out)
        for i in range(n):
            for j in range(cfg.layers_per_block + 1):
                x = self._s_res(x, f"s.up.{i}.resnets.{j}",
                                stats_out=i == n - 1 or j < cfg.layers_per_block)
            if i < n - 1:
                B, T, H, Wd, C = x.shape
                up = torch.empty((B, T, 2 * H, 2 * Wd, C), dtype=torch.bfloat16, device=self.dev)
                check(lib().ddit_upsample2x(ptr(x), ptr(up), B * T, H, Wd, C, stream_ptr()))
                self.launches += 1
                x = self._conv(up, f"s.up.{i}.upsample", causal=False, gn_stats=True)
        x = self._gn(x, "s.norm_out", cfg.sd_eps, per_frame=True)
        y = self._conv(x, "s.conv_out", causal=False, pad_bias=True)  # [N, 1, H, W, 64]
        B, T, H, Wd, C = y.shape
        # channels-first fp32 frames, 3 valid channels, cropped to (height, width)
        frames = torch.empty((1, 3, N, height, width), dtype=torch.float32, device=self.dev)
        check(lib().ddit_frames_out(ptr(y), ptr(frames), N, H, Wd, C, 3, height, width, stream_ptr()))
        self.launches += 1
        return frames

    # ---------------------------------------------------------------- pipeline
    def decode(self, z: torch.Tensor, num_frames: int, height: int, width: int,
               frames: tuple[int, int] | None = None) -> torch.Tensor:
        """The decode below, replayed from a CUDA graph once a shape has been seen: the first call
        per (latent shape, frames, size) runs eagerly and captures; later calls copy z into the
        graph's input and replay its ~850 launches as one (LRU of ``graphs`` shapes; the graph
        pool keeps that shape's activations resident). Same kernels, same bits as eager."""
        if self.max_graphs <= 0:
            return self.decode_eager(z, num_frames, height, width, frames)
        key = (tuple(z.shape), tuple(z.stride()), num_frames, height, width, frames)
        ent = self._graphs.pop(key, None)
        if ent is None:
            out = self.decode_eager(z, num_frames, height, width, frames)  # also the warm-up
            static_z = z.clone()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                static_out = self.decode_eager(static_z, num_frames, height, width, frames)
            self._graphs[key] = (g, static_z, static_out)
            while len(self._graphs) > self.max_graphs:
                self._graphs.pop(next(iter(self._graphs)))
            return out
        g, static_z, static_out = ent
        self._graphs[key] = ent  # most recent last
        static_z.copy_(z)
        g.replay()
        return static_out.clone()

    def decode_eager(self, z: torch.Tensor, num_frames: int, height: int, width: int,
                     frames: tuple[int, int] | None = None) -> torch.Tensor:
        """VideoAutoencoderPipeline.decode: z [1, 4, T, h, w] fp32 (device) ->
        video [1, 3, num_frames, height, width] fp32. ``frames=(a, b)``: only video frames
        [a, b) of the ``num_frames`` that z's micro-batches decode to (VAE DoP, ``vae_shard``)."""
        cfg = self.cfg
        assert z.shape[0] == 1 and z.is_cuda
        parts = []
        left = num_frames
        for t0 in range(0, z.shape[2], cfg.micro_z):
            t1 = min(t0 + cfg.micro_z, z.shape[2])
            parts.append(self.temporal_decode(z, t0, t1, min(cfg.micro_frame_size, left)))
            left -= cfg.micro_frame_size
        x4 = torch.cat(parts, dim=1) if len(parts) > 1 else parts[0]
        if frames is not None:
            x4 = x4[:, frames[0]:frames[1]]
        return self.spatial_decode(x4.contiguous(), height, width)


def vae_shard(cfg: VAEConfig, t_latent: int, frames: int, dop: int, rank: int) -> tuple[int, int, int, int]:
    """VAE DoP: rank ``rank`` of ``dop`` produces the contiguous video frames [f_lo, f_hi)
    (ceil(frames / dop) each). The spatial decoder (81 % of the decode FLOPs at 240p) is per frame
    and the temporal VAE decodes its micro-batches (``micro_z`` latent frames ->
    ``micro_frame_size`` video frames) independently (VideoAutoencoderPipeline.decode), so a rank
    temporal-decodes the micro-batches its frames fall in -- latent [t_lo, t_hi), duplicating at
    most one boundary micro-batch of cheap temporal work -- and spatially decodes only its own
    frames: no halo exchange, and the ranks' frames concatenate to the DoP-1 video exactly.
    Returns (t_lo, t_hi, f_lo, f_hi); empty ranges have lo == hi."""
    per = -(-frames // dop)
    f_lo, f_hi = min(rank * per, frames), min((rank + 1) * per, frames)
    if f_hi <= f_lo:
        return t_latent, t_latent, frames, frames
    c_lo, c_hi = f_lo // cfg.micro_frame_size, -(-f_hi // cfg.micro_frame_size)
    return (c_lo * cfg.micro_z, min(c_hi * cfg.micro_z, t_latent), f_lo, f_hi)


def vae_flops(cfg: VAEConfig, frames: int, t_latent: int, h: int, w: int) -> float:
    """Algorithmic FLOPs of one decode (tensor-core convs + attention), for the roofline."""
    fl = 0.0

    def conv(cin, cout, k, pix):
        nonlocal fl
        fl += 2.0 * k * cin * cout * pix

    # temporal, per micro chunk
    chunks = -(-t_latent // cfg.micro_z)
    top = cfg.t_filters * cfg.t_mults[-1]
    for c in range(chunks):
        T = min(cfg.micro_z, t_latent - c * cfg.micro_z)
        pix = T * h * w
        conv(4, top, 27, pix)
        for _ in range(cfg.t_res_blocks):
            conv(top, top, 27, pix)
            conv(top, top, 27, pix)
        prev = top
        for i in reversed(range(len(cfg.t_mults))):
            f = cfg.t_filters * cfg.t_mults[i]
            for j in range(cfg.t_res_blocks):
                conv(prev, f, 27, pix)
                conv(f, f, 27, pix)
                if prev != f:
                    conv(prev, f, 1, pix)
                prev = f
            if i > 0 and cfg.t_downsample[i - 1]:
                conv(prev, 2 * prev, 27, pix)
                pix *= 2
        conv(prev, 4, 27, pix)
    # spatial, per frame
    rev = list(reversed(cfg.block_out))
    pix = frames * h * w
    conv(4, rev[0], 9, pix)
    for _ in range(2):
        conv(rev[0], rev[0], 9, pix)
        conv(rev[0], rev[0], 9, pix)
    fl += 4.0 * frames * (h * w) ** 2 * rev[0] + 8.0 * pix * rev[0] ** 2
    prev = rev[0]
    for i, ch in enumerate(rev):
        for j in range(cfg.layers_per_block + 1):
            conv(prev, ch, 9, pix)
            conv(ch, ch, 9, pix)
            if prev != ch:
                conv(prev, ch, 1, pix)
            prev = ch
        if i < len(rev) - 1:
            pix *= 4
            conv(ch, ch, 9, pix)
    conv(prev, 3, 9, pix)
    return fl
