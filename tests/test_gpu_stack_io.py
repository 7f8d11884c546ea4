"""Slice-stack decode + normalisation on the device (vk_decode_samples /
vk_normalize_stack through the C ABI) against the live reference's stacks
(tests/golden/reference_stack.npz) and the numpy oracle: bit-exact."""

import json
import os

import numpy as np
import pytest

from oracle import stack_oracle as SO

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.realpath(os.path.join(HERE, "golden"))


def _bits_equal(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_load_stack_matches_reference(cuda):
    from paper_2303_09523_b200 import load_stack
    blob = np.load(os.path.join(GOLD, "reference_stack.npz"))
    with open(os.path.join(GOLD, "reference_stack.json")) as f:
        meta = json.load(f)
    for s in meta["stacks"]:
        st = load_stack(os.path.join(GOLD, s["manifest"]), device=True)
        assert st.on_device and st.slices.is_cuda
        assert _bits_equal(st.slices.cpu().numpy(), blob[f"{s['name']}/slices"]), s["name"]
        host = load_stack(os.path.join(GOLD, s["manifest"]), device=False)
        assert isinstance(host.slices, np.ndarray) and _bits_equal(host.slices, blob[f"{s['name']}/slices"])
        assert host.pixel_spacing == tuple(s["pixel_spacing"]) and host.axis_label == s["axis_label"]


@pytest.mark.parametrize("kind,dtype,lo,hi", [(0, np.uint8, 0, 256), (1, np.uint16, 0, 65536),
                                              (2, np.int32, -2 ** 31, 2 ** 31 - 1)])
def test_decode_samples_all_types(cuda, kind, dtype, lo, hi):
    torch = cuda
    from paper_2303_09523_b200.stack_io import decode_samples
    r = np.random.default_rng(kind)
    raw = r.integers(lo, hi, size=(3, 37, 41), dtype=np.int64).astype(dtype)
    if kind == 2:   # values above 2^24 exercise the int -> f32 rounding
        raw.flat[:6] = [2 ** 24 + 1, 2 ** 24 + 3, -(2 ** 24 + 1), 2 ** 31 - 1, -2 ** 31, 0]
    dev = torch.from_numpy(raw.view(np.uint8)).cuda()
    got = decode_samples(dev, kind).view(raw.shape).cpu().numpy()
    exp = SO.decode(raw, 255.0 if kind == 0 else 65535.0)
    assert _bits_equal(got, exp)


@pytest.mark.parametrize("kind,dtype,top", [(0, np.uint8, 255), (1, np.uint16, 4095), (1, np.uint16, 65535),
                                            (2, np.int32, 70000)])
def test_normalize_raw_samples(cuda, kind, dtype, top):
    torch = cuda
    from paper_2303_09523_b200.stack_io import _normalize_dev
    r = np.random.default_rng(top)
    raw = (r.integers(0, top + 1, size=(5, 64, 80)) + (7 if top < 255 else 0)).astype(dtype)
    dev = torch.from_numpy(raw.view(np.uint8)).cuda()
    got = _normalize_dev(dev, kind).view(raw.shape).cpu().numpy()
    exp = SO.normalize(SO.decode(raw, 255.0 if kind == 0 else 65535.0))
    assert _bits_equal(got, exp)


def test_normalize_stack_f32(cuda):
    torch = cuda
    from paper_2303_09523_b200 import SliceStack
    from paper_2303_09523_b200.stack_io import normalize_stack
    r = np.random.default_rng(189)
    for data in (r.normal(3.0, 2.0, size=(4, 33, 29)).astype(np.float32),
                 (r.random((3, 16, 16)) * 1e-30 + 1.0).astype(np.float32),
                 np.concatenate([np.full((1, 8, 8), -1e30, np.float32), np.full((1, 8, 8), 1e-30, np.float32),
                                 r.normal(size=(1, 8, 8)).astype(np.float32)]),
                 np.full((2, 5, 6), -4.25, np.float32)):
        exp = SO.normalize(data)
        for src in (data, torch.from_numpy(data).cuda()):
            st = normalize_stack(SliceStack(src, (1.0, 1.0), 2.0))
            assert st.on_device and _bits_equal(st.slices.cpu().numpy(), exp)


def test_normalize_full_size_u16(cuda):
    """C5-sized raw stack (512 x 1024^2 u16, 1 GiB) normalised on the device,
    checked against numpy on a strided sample plus the exact extremes."""
    torch = cuda
    from paper_2303_09523_b200.stack_io import SAMPLE_U16, _normalize_dev
    g = torch.Generator(device="cuda").manual_seed(5)
    raw = torch.randint(100, 60001, (512, 1024, 1024), device="cuda", generator=g, dtype=torch.int32)
    raw[17, 3, 5] = 99
    raw[400, 1000, 1023] = 60001
    raw16 = torch.where(raw > 32767, raw - 65536, raw).to(torch.int16)   # bit pattern of the u16 samples
    del raw
    out = _normalize_dev(raw16, SAMPLE_U16).view(raw16.shape)
    assert float(out.min()) == 0.0 and float(out.max()) == 1.0
    assert float(out[17, 3, 5]) == 0.0 and float(out[400, 1000, 1023]) == 1.0
    idx = torch.arange(0, out.numel(), 7919, device="cuda")
    samp = raw16.view(-1)[idx].cpu().numpy().view(np.uint16)
    lo = np.float32(99) / np.float32(65535.0)
    hi = np.float32(60001) / np.float32(65535.0)
    exp = (SO.decode(samp, 65535.0) - lo) / np.float32(float(hi) - float(lo))
    assert _bits_equal(out.view(-1)[idx].cpu().numpy(), exp)


@pytest.mark.parametrize("kind,dtype", [(0, np.uint8), (1, np.uint16), (2, np.int32), (3, np.float32)])
def test_unaligned_buffers_and_tails(cuda, kind, dtype):
    """16-byte-vector body + scalar tail, and the scalar path for buffers that
    are not 16-byte aligned (raw or out), in place for f32."""
    torch = cuda
    from paper_2303_09523_b200 import _lib
    from paper_2303_09523_b200.kriging import _stream_handle
    lib = _lib.load()
    r = np.random.default_rng(31 + kind)
    scale = 255.0 if kind == 0 else 65535.0
    for n in (1, 3, 5, 17, 63, 1000003):
        if kind == 3:
            raw = r.normal(size=n + 1).astype(np.float32)
        else:
            info = np.iinfo(dtype)
            raw = r.integers(max(info.min, -10 ** 6), min(info.max, 10 ** 6), size=n + 1, endpoint=True).astype(dtype)
        dev = torch.from_numpy(raw.view(np.uint8).copy()).cuda()
        isz = raw.itemsize
        for off, out_off in ((0, 0), (1, 0), (0, 1), (1, 1)):
            out = torch.full((n + 1,), -7.0, dtype=torch.float32, device="cuda")
            src = raw[off:off + n]
            dec = SO.decode(src, scale) if kind != 3 else src
            assert lib.vk_decode_samples(dev.data_ptr() + off * isz, kind, n, out.data_ptr() + 4 * out_off,
                                         _stream_handle(None)) == 0
            got = out.cpu().numpy()
            assert _bits_equal(got[out_off:out_off + n], dec), (n, off, out_off)
            assert got[1 - out_off if out_off else n] == -7.0        # no write past the range
            assert lib.vk_normalize_stack(dev.data_ptr() + off * isz, kind, n, out.data_ptr() + 4 * out_off,
                                          None, _stream_handle(None)) == 0
            assert _bits_equal(out.cpu().numpy()[out_off:out_off + n], SO.normalize(dec)), (n, off, out_off)
        if kind == 3:          # in place
            buf = torch.from_numpy(raw.copy()).cuda()
            assert lib.vk_normalize_stack(buf.data_ptr() + 4, 3, n, buf.data_ptr() + 4, None,
                                          _stream_handle(None)) == 0
            got = buf.cpu().numpy()
            assert got[0] == raw[0] and _bits_equal(got[1:], SO.normalize(raw[1:]))


def test_formats_around_the_path(cuda, tmp_path):
    """load_stack -> Z-part kriging -> save_volume -> load_volume, all on the
    device, against the oracle pipeline on the reference's own stack."""
    from oracle import kriging_oracle as O
    from paper_2303_09523_b200 import VolumeGrid, ZPartKriging, load_stack, load_volume, save_volume
    blob = np.load(os.path.join(GOLD, "reference_stack.npz"))
    st = load_stack(os.path.join(GOLD, "stack", "u8_L", "stack.manifest"), device=True)
    assert st.factor == 3 and st.output_depth() == 10
    zk = ZPartKriging(st.n, st.height, st.width, st.factor, 1)
    vol, _ = zk.run(st.slices)
    zk.finish()
    ref, _, _ = O.reconstruct_zparts(blob["u8_L/slices"], st.factor, 1)
    assert np.abs(vol.cpu().numpy().astype(np.float64) - ref).max() <= 1e-6 * 1.0   # normalised range is 1
    path = tmp_path / "out.vkv"
    save_volume(VolumeGrid(vol), path)
    back = load_volume(path, device=True)
    assert _bits_equal(back.data.cpu().numpy(), vol.cpu().numpy()) and not bool(back.missing_mask.any())
