"""Numerics check behind a design decision: how far does a bf16 residual
stream (x rounded to bf16 after every residual add, everything else fp32) move one XL/2 denoise
step away from the fp32 oracle? CPU only. Usage: python scripts/bf16_residual_numerics.py [144p]"""
import sys, time, torch, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import stdit3
from paper_2506_13497_b200 import weights, shapes
torch.set_num_threads(os.cpu_count())
label = sys.argv[1] if len(sys.argv) > 1 else "144p"
cfg = weights.XL2
W = weights.init_weights(cfg, seed=3)
sh = shapes.shape_of(label)
z, y = weights.synthetic_inputs(cfg, sh.latent)
text = stdit3.prepare_text(W, y)
orig_block = stdit3.block
F = torch.nn.functional
def rb(t): return t.to(torch.bfloat16).float()
def block_bf16res(W, cfg, kind, i, x, y, t_mlp, T, S):
    p = f"{kind}_blocks.{i}."
    B, N, C = x.shape
    mod = W[p + "scale_shift_table"][None] + t_mlp.view(B, 6, C)
    shift_msa, scale_msa, gate_msa, shift_mlp, scale_mlp, gate_mlp = mod.unbind(1)
    xm = stdit3.layer_norm(x, cfg.eps) * (1 + scale_msa[:, None]) + shift_msa[:, None]
    if kind == "temporal":
        xs = xm.view(B, T, S, C).transpose(1, 2).reshape(B * S, T, C)
        o = stdit3.self_attention(W, p, cfg, xs, rope=True)
        o = o.view(B, S, T, C).transpose(1, 2).reshape(B, N, C)
    else:
        xs = xm.view(B * T, S, C)
        o = stdit3.self_attention(W, p, cfg, xs, rope=False).view(B, N, C)
    x = rb(x + rb(gate_msa[:, None] * o))
    x = rb(x + rb(stdit3.cross_attention(W, p, cfg, x, y)))
    xm = stdit3.layer_norm(x, cfg.eps) * (1 + scale_mlp[:, None]) + shift_mlp[:, None]
    h = F.gelu(F.linear(xm, W[p + "mlp.fc1.weight"], W[p + "mlp.fc1.bias"]), approximate="tanh")
    h = F.linear(h, W[p + "mlp.fc2.weight"], W[p + "mlp.fc2.bias"])
    return rb(x + rb(gate_mlp[:, None] * h))
def rel(a, b): return (torch.linalg.vector_norm(a-b)/torch.linalg.vector_norm(b)).item()
with torch.inference_mode():
    for step in (3, 20):
        t0=time.time()
        ref = stdit3.denoise_step(W, cfg, z, text, step, sh.height, sh.width)
        stdit3.block = block_bf16res
        out = stdit3.denoise_step(W, cfg, z, text, step, sh.height, sh.width)
        stdit3.block = orig_block
        print(label, "step", step, "bf16-residual vs fp32: z'", f"{rel(out, ref):.2e}", "update", f"{rel(out-z, ref-z):.2e}", f"{time.time()-t0:.0f}s", flush=True)
