"""Binary volume format on the device (io.py:146-200): CRC-32 against zlib,
bit packing against numpy, byte-identical files against the ones the live
reference wrote, CRC corruption detection, large round trips."""

import os
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("n", [0, 1, 3, 15, 16, 17, 100, 16383, 16384, 16385, 1_000_003, 50_000_017])
def test_crc32_matches_zlib(cuda, n):
    torch = cuda
    from paper_2303_09523_b200.volume_io import crc32
    r = np.random.default_rng(n)
    buf = r.integers(0, 256, n + 5, dtype=np.uint8)
    d = torch.from_numpy(buf).cuda()
    for off in (0, 1, 5):                               # unaligned starts
        seg = buf[off:off + n]
        for c0 in (0, 0xDEADBEEF, zlib.crc32(b"VOLKRIG")):
            assert crc32(d[off:off + n], len(seg), c0) == zlib.crc32(seg.tobytes(), c0)


@pytest.mark.parametrize("n", [1, 7, 8, 9, 63, 64, 65, 1000, 1_048_577])
def test_packbits_roundtrip(cuda, n):
    torch = cuda
    from paper_2303_09523_b200.volume_io import packbits, unpackbits
    m = np.random.default_rng(n).random(n) < 0.3
    bits = packbits(torch.from_numpy(m).cuda())
    assert np.array_equal(bits.cpu().numpy(), np.packbits(m))
    back = unpackbits(bits, n)
    assert np.array_equal(back.cpu().numpy(), m)


@pytest.mark.parametrize("key", ["a", "b", "c"])
@pytest.mark.parametrize("on_device", [False, True])
def test_save_is_byte_identical_to_reference(cuda, tmp_path, key, on_device):
    torch = cuda
    from paper_2303_09523_b200 import VolumeGrid
    from paper_2303_09523_b200.volume_io import save_volume
    g = np.load(os.path.join(HERE, "golden", "reference_volio.npz"))
    d, m, o = g[f"{key}/data"], g[f"{key}/mask"], tuple(int(v) for v in g[f"{key}/origin"])
    grid = VolumeGrid(torch.from_numpy(d).cuda(), torch.from_numpy(m).cuda(), o) if on_device \
        else VolumeGrid(d, m, o)
    p = tmp_path / f"{key}.vkv"
    save_volume(grid, p)
    with open(os.path.join(HERE, "golden", f"ref_volume_{key}.vkv"), "rb") as f:
        assert p.read_bytes() == f.read()


@pytest.mark.parametrize("key", ["a", "b", "c"])
def test_load_reference_files(cuda, key):
    from paper_2303_09523_b200.volume_io import load_volume
    g = np.load(os.path.join(HERE, "golden", "reference_volio.npz"))
    path = os.path.join(HERE, "golden", f"ref_volume_{key}.vkv")
    for device in (True, False):
        v = load_volume(path, device=device)
        data = v.data.cpu().numpy() if device else v.data
        mask = v.missing_mask.cpu().numpy() if device else v.missing_mask
        assert np.array_equal(mask, g[f"{key}/mask"])
        assert np.array_equal(data, g[f"{key}/data"], equal_nan=True)
        assert v.origin_offset == tuple(int(x) for x in g[f"{key}/origin"])


def test_crc_corruption_detected(cuda, tmp_path):
    from paper_2303_09523_b200.errors import ChecksumMismatch
    from paper_2303_09523_b200.volume_io import load_volume
    with open(os.path.join(HERE, "golden", "ref_volume_a.vkv"), "rb") as f:
        b = bytearray(f.read())
    for pos in (40, len(b) - 10, len(b) - 2):          # payload, mask, stored CRC
        c = bytearray(b)
        c[pos] ^= 0x10
        p = tmp_path / f"bad{pos}.vkv"
        p.write_bytes(bytes(c))
        with pytest.raises(ChecksumMismatch):
            load_volume(p, device=True)


def test_large_round_trip(cuda, tmp_path):
    torch = cuda
    from paper_2303_09523_b200 import VolumeGrid
    from paper_2303_09523_b200.volume_io import load_volume, save_volume
    r = np.random.default_rng(9)
    d = r.normal(size=(33, 256, 256)).astype(np.float32)
    m = r.random(d.shape) < 0.5
    d[m] = np.nan
    p = tmp_path / "big.vkv"
    save_volume(VolumeGrid(torch.from_numpy(d).cuda(), torch.from_numpy(m).cuda(), (3, 2, 1)), p)
    raw = p.read_bytes()
    assert zlib.crc32(raw[:-4]) == int.from_bytes(raw[-4:], "little")
    v = load_volume(p, device=True)
    assert torch.equal(v.missing_mask.cpu(), torch.from_numpy(m))
    assert np.array_equal(v.data.cpu().numpy(), d, equal_nan=True)


def test_plan_download_regular_and_irregular(cuda):
    """vk_plan_download: interpolated planes from the device, known planes
    from the host input -- the same bytes as a full device-to-host copy."""
    torch = cuda
    from paper_2303_09523_b200 import ZPartKriging
    from paper_2303_09523_b200.kriging import KrigingPlan, VariogramModel
    from paper_2303_09523_b200.phantoms import known_slices, small_config
    cfg = small_config("spine", 40, 52, 9, 4, n_subparts=2, seed=3)
    ks = known_slices(cfg)
    zk = ZPartKriging(cfg.n_known, cfg.height, cfg.width, cfg.factor, cfg.n_subparts)
    out, _ = zk.run(torch.from_numpy(ks).cuda())
    host = zk.download(out, torch.from_numpy(ks).pin_memory())
    zk.finish()
    assert host.is_pinned() and torch.equal(host, out.cpu())
    # irregular known planes (runs of 1, 2, 3 and 4 missing planes)
    kz = np.array([0, 2, 5, 9, 10, 15], np.int32)
    T, H, W = 16, 24, 28
    r = np.random.default_rng(4)
    known = (r.random((len(kz), H, W)) * 100).astype(np.float32)
    plan = KrigingPlan(H, W, T, kz, fit=False)
    m = VariogramModel("exponential", 0.5, 500.0, 6.0)
    outd = torch.full((T, H, W), float("nan"), device="cuda")
    plan.execute(torch.from_numpy(known).cuda(), outd, models=np.array([[m.nugget, m.sill, m.range_len]]))
    h2 = plan.download(outd, torch.from_numpy(known))
    plan.finish()
    ref = outd.cpu()
    assert torch.equal(h2[kz], torch.from_numpy(known))
    miss = np.setdiff1d(np.arange(T), kz)
    assert torch.equal(h2[miss].view(torch.int32), ref[miss].view(torch.int32))
