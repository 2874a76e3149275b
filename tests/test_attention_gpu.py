"""Flash attention (spatial / temporal / cross index maps) vs torch fp32 softmax attention."""
import pytest
import torch

pytestmark = pytest.mark.gpu
H, D = 16, 72


def rel_l2(a, b):
    return (torch.linalg.vector_norm(a.float() - b.float()) / torch.linalg.vector_norm(b.float())).item()


def ref_attn(q, k, v):  # [n, L, H, D]
    s = torch.einsum("nqhd,nkhd->nhqk", q.float(), k.float()) * D**-0.5
    return torch.einsum("nhqk,nkhd->nqhd", s.softmax(-1), v.float())


@pytest.mark.parametrize("B,T,S", [(2, 3, 405), (2, 1, 64), (1, 2, 130), (2, 4, 1), (2, 2, 920), (1, 1, 1620), (1, 3, 256),
                                   (2, 1, 3600), (1, 2, 3600)])
def test_spatial(cuda, B, T, S):
    from paper_2506_13497_b200 import kernels
    g = torch.Generator().manual_seed(0)
    M = B * T * S
    qkv = torch.randn(M, 3 * H * D, generator=g).to(cuda, torch.bfloat16)
    o = torch.zeros(M, H * D, device=cuda, dtype=torch.bfloat16)
    C = H * D
    kernels.attention(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], o, heads=H, num_seqs=B * T,
                      Lq=S, Lk=S, q_map=(1, S, 0, 1), kv_map=(1, S, 0, 1))
    q, k, v = qkv.view(B * T, S, 3, H, D).unbind(2)
    ref = ref_attn(q, k, v).reshape(M, C)
    e = rel_l2(o, ref)
    print(f"spatial B={B} T={T} S={S}: relL2 {e:.2e}")
    assert e < 1e-2


@pytest.mark.parametrize("B,T,Sl", [(2, 15, 405), (2, 30, 17), (1, 4, 3), (2, 16, 9), (1, 32, 2), (2, 1, 3),
                                    (2, 30, 450), (2, 60, 37), (1, 45, 9), (1, 64, 5)])
def test_temporal(cuda, B, T, Sl):
    from paper_2506_13497_b200 import kernels
    g = torch.Generator().manual_seed(1)
    M = B * T * Sl
    C = H * D
    qkv = torch.randn(M, 3 * C, generator=g).to(cuda, torch.bfloat16)
    o = torch.zeros(M, C, device=cuda, dtype=torch.bfloat16)
    mp = (Sl, T * Sl, 1, Sl)
    kernels.attention(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], o, heads=H, num_seqs=B * Sl,
                      Lq=T, Lk=T, q_map=mp, kv_map=mp, temporal=True)
    x = qkv.view(B, T, Sl, 3, H, D).transpose(1, 2).reshape(B * Sl, T, 3, H, D)
    q, k, v = x.unbind(2)
    ref = ref_attn(q, k, v).reshape(B, Sl, T, C).transpose(1, 2).reshape(M, C)
    e = rel_l2(o, ref)
    print(f"temporal B={B} T={T} Sl={Sl}: relL2 {e:.2e}")
    assert e < 1e-2


@pytest.mark.parametrize("heads", [4, 12, 20])
@pytest.mark.parametrize("T", [15, 30, 60])
def test_temporal_head_counts(cuda, heads, T):
    """The tcgen05 temporal kernel stacks 128 / R heads per tile (8 at T <= 16, 4 at T <= 32):
    head counts below one group (4 at T=15), and a partial last group (12, 20 at T=15; none at
    T=30), against torch fp32."""
    from paper_2506_13497_b200 import kernels
    g = torch.Generator().manual_seed(3)
    B, Sl = 2, 37
    C = heads * D
    M = B * T * Sl
    qkv = torch.randn(M, 3 * C, generator=g).to(cuda, torch.bfloat16)
    o = torch.full((M, C), float("nan"), device=cuda, dtype=torch.bfloat16)
    mp = (Sl, T * Sl, 1, Sl)
    kernels.attention(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], o, heads=heads, num_seqs=B * Sl,
                      Lq=T, Lk=T, q_map=mp, kv_map=mp, temporal=True)
    x = qkv.view(B, T, Sl, 3, heads, D).transpose(1, 2).reshape(B * Sl, T, 3, heads, D)
    q, k, v = x.unbind(2)
    ref = ref_attn(q, k, v).reshape(B, Sl, T, C).transpose(1, 2).reshape(M, C)
    assert not torch.isnan(o).any()
    assert rel_l2(o, ref) < 1e-2


@pytest.mark.parametrize("B,N,Ly", [(2, 777, 300), (2, 64, 300), (1, 100, 17), (2, 6075, 300)])
def test_cross(cuda, B, N, Ly):
    from paper_2506_13497_b200 import kernels
    g = torch.Generator().manual_seed(2)
    C = H * D
    q = torch.randn(B * N, C, generator=g).to(cuda, torch.bfloat16)
    kv = torch.randn(B * Ly, 2 * C, generator=g).to(cuda, torch.bfloat16)
    o = torch.zeros(B * N, C, device=cuda, dtype=torch.bfloat16)
    kernels.attention(q, kv[:, :C], kv[:, C:], o, heads=H, num_seqs=B, Lq=N, Lk=Ly,
                      q_map=(1, N, 0, 1), kv_map=(1, Ly, 0, 1))
    kk, vv = kv.view(B, Ly, 2, H, D).unbind(2)
    ref = ref_attn(q.view(B, N, H, D), kk, vv).reshape(B * N, C)
    assert rel_l2(o, ref) < 1e-2


def test_tc_large_logits_rescale(cuda):
    """Scores growing along the key axis force the lazy O rescale path."""
    from paper_2506_13497_b200 import kernels
    B, T, S = 1, 2, 700
    C = H * D
    g = torch.Generator().manual_seed(5)
    qkv = torch.randn(B * T * S, 3 * C, generator=g)
    ramp = torch.linspace(0, 6, S).repeat(B * T)[:, None]
    qkv[:, C:2 * C] *= ramp  # later keys -> much larger logits
    qkv = qkv.to(cuda, torch.bfloat16)
    o = torch.zeros(B * T * S, C, device=cuda, dtype=torch.bfloat16)
    kernels.attention(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], o, heads=H, num_seqs=B * T,
                      Lq=S, Lk=S, q_map=(1, S, 0, 1), kv_map=(1, S, 0, 1), tc=True)
    q, k, v = qkv.view(B * T, S, 3, H, D).unbind(2)
    ref = ref_attn(q, k, v).reshape(B * T * S, C)
    assert rel_l2(o, ref) < 1e-2
