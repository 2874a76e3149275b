"""On-disk latent / frames format (paper_2506_13497_b200.latent_io): exact round trips, header
fields, payload alignment and corruption detection."""
import pytest
import torch

from paper_2506_13497_b200.latent_io import ALIGN, LatentFormatError, load_latent, save_latent


def test_round_trip_latent_and_frames(tmp_path):
    g = torch.Generator().manual_seed(0)
    z = torch.randn(1, 4, 15, 30, 54, generator=g)
    fr = torch.randint(0, 256, (51, 240, 426, 3), generator=g, dtype=torch.uint8)
    p = tmp_path / "r7.ddlat"
    n = save_latent(p, z, request_id=7, resolution="240p", steps=30, frames=fr, dop=4)
    assert p.stat().st_size == n
    z2, f2, h = load_latent(p)
    assert torch.equal(z2, z) and torch.equal(f2, fr)
    assert h["request_id"] == 7 and h["resolution"] == "240p" and h["dop"] == 4
    assert h["shape"] == [1, 4, 15, 30, 54]
    raw = p.read_bytes()
    assert (n - h["payload_bytes"] - h["frames_bytes"]) % ALIGN == 0


def test_bf16_latent_without_frames(tmp_path):
    z = torch.randn(2, 3, 5).to(torch.bfloat16)
    p = tmp_path / "a.ddlat"
    save_latent(p, z, request_id=1, resolution="144p", steps=1)
    z2, f2, h = load_latent(p)
    assert f2 is None and h["dtype"] == "bf16" and torch.equal(z2, z)


def test_corruption_is_detected(tmp_path):
    z = torch.randn(1, 4, 2, 3, 3)
    p = tmp_path / "c.ddlat"
    save_latent(p, z, request_id=0, resolution="144p", steps=3)
    raw = bytearray(p.read_bytes())
    raw[-1] ^= 1
    p.write_bytes(bytes(raw))
    with pytest.raises(LatentFormatError, match="checksum"):
        load_latent(p)
    p.write_bytes(bytes(raw[:-5]))
    with pytest.raises(LatentFormatError, match="truncated"):
        load_latent(p)
    p.write_bytes(b"NOTALATENTFILE")
    with pytest.raises(LatentFormatError, match="magic"):
        load_latent(p)
