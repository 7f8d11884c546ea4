"""The streaming kernel's guided dynamic unit schedule (vk_predict.cu,
FtSched): units are claimed from a global counter in an order that depends on
timing, so the same launch must (a) write every voxel, (b) give bit-identical
volumes run after run, and (c) agree bit for bit with the per-part chained
launches, which cut the same gaps into different units (one level, half a
part's gaps).  Shapes are chosen so the serial launch has several levels
(10 / 5 / 2 / 1-gap units) and many more units than resident CTAs.
(kriging.py:499-557 is the path; the values themselves are checked against
the oracle in test_gpu_parity.py / test_gpu_fullsize.py.)
"""

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu]


def _planes(shape, seed, integer):
    r = np.random.default_rng(seed)
    K, H, W = shape
    z = np.arange(K, dtype=np.float32)[:, None, None]
    y = np.arange(H, dtype=np.float32)[None, :, None]
    x = np.arange(W, dtype=np.float32)[None, None, :]
    base = 900.0 + 300.0 * np.sin(0.11 * x + 0.07 * y) * np.cos(0.05 * z) + 0.8 * z
    v = base + r.normal(0.0, 25.0, size=shape)
    if integer:
        return np.clip(np.rint(v), 0, 4095).astype(np.float32)
    return (v / 4095.0).astype(np.float32)


@pytest.mark.parametrize("shape,factor,parts,accum,integer", [
    ((256, 128, 384), 8, 32, "fp64", True),     # exact-split rows, G = 7, 12 tiles x 255 gaps
    ((256, 128, 384), 8, 32, "fp64", False),    # 16-tap DFMA rows
    ((128, 96, 256), 4, 16, "fp32", False),     # G = 3: three CTAs per SM, 3-deep ring
    ((40, 70, 132), 2, 5, "fp64", True),        # G = 1, ragged tile edges, uneven parts
    ((5, 24, 64), 4, 4, "fp64", True),          # one gap per part, all border rows in one tile
    ((9, 30, 64), 8, 8, "fp64", False),         # same with G = 7
])
def test_guided_schedule_complete_deterministic_and_equal_to_chains(cuda, shape, factor, parts, accum, integer):
    torch = cuda
    from paper_2303_09523_b200 import ZPartKriging
    K, H, W = shape
    ks = torch.from_numpy(_planes(shape, 5, integer)).cuda()
    serial = ZPartKriging(K, H, W, factor, parts, accum=accum, overlap=False)
    chained = ZPartKriging(K, H, W, factor, parts, accum=accum, overlap=True)
    out, var = serial.allocate(True)
    ref = ref_var = None
    for rep in range(5):
        out.fill_(float("nan"))
        var.fill_(float("nan"))
        serial.run(ks, out, var)
        serial.finish()
        assert not bool(torch.isnan(out).any()), "a unit of the schedule was never run"
        assert not bool(torch.isnan(var).any())
        if ref is None:
            ref, ref_var = out.clone(), var.clone()
        else:
            assert torch.equal(out, ref), f"run {rep} differs from run 0"
            assert torch.equal(var, ref_var)
    # known planes pass through bit-exactly
    assert torch.equal(ref[::factor], ks)
    out2, var2 = chained.allocate(True)
    out2.fill_(float("nan"))
    var2.fill_(float("nan"))
    chained.run(ks, out2, var2)
    chained.finish()
    assert torch.equal(out2, ref), "per-part chained launches differ from the serial launch"
    assert torch.equal(var2, ref_var)


def test_guided_schedule_without_variance_back_to_back(cuda):
    """Back-to-back launches of one plan without a host sync in between: the
    last CTA of a launch rewinds the unit counter for the next."""
    torch = cuda
    from paper_2303_09523_b200 import ZPartKriging
    shape, factor, parts = (256, 64, 256), 8, 32
    K, H, W = shape
    ks = torch.from_numpy(_planes(shape, 9, True)).cuda()
    zk = ZPartKriging(K, H, W, factor, parts, overlap=False)
    outs = [zk.allocate(False)[0] for _ in range(4)]
    for o in outs:
        o.fill_(float("nan"))
    for o in outs:
        zk.run(ks, o)
    zk.finish()
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    assert not bool(torch.isnan(outs[0]).any())
