"""LayerNorm + t2i-modulate kernel against a torch fp32 reference, through
the C ABI, for the step's C = 1152 variants and the generic width path."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("variant", [1, 3])
@pytest.mark.parametrize("M,C,nb", [(12150, 1152, 2), (1519, 1152, 2), (37, 1152, 3), (300, 288, 2)])
def test_ln_modulate_matches_torch(cuda, variant, M, C, nb):
    from paper_2506_13497_b200 import _lib

    L = _lib.lib()
    g = torch.Generator(device=cuda).manual_seed(M + C)
    x = 3 * torch.randn(M, C, device=cuda, generator=g) + 0.5
    mods = torch.randn(nb, 6, C, device=cuda, generator=g)
    shift, scale = mods[:, 0], mods[:, 1]
    rpb = -(-M // nb)
    out = torch.empty(M, C, device=cuda, dtype=torch.bfloat16)
    try:
        _lib.check(L.ddit_set_ln_variant(variant))
        _lib.check(L.ddit_ln_modulate(x.data_ptr(), out.data_ptr(), M, C, shift.data_ptr(),
                                      scale.data_ptr(), 6 * C, rpb, 1e-6,
                                      torch.cuda.current_stream().cuda_stream))
    finally:
        L.ddit_set_ln_variant(3)
    torch.cuda.synchronize()
    b = torch.arange(M, device=cuda) // rpb
    ref = torch.nn.functional.layer_norm(x, (C,), eps=1e-6) * (1 + scale[b]) + shift[b]
    err = ((out.float() - ref).norm() / ref.norm()).item()
    assert err < 4e-3, err
