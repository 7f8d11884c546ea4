"""GPU parity of the shipped path (device fit -> solve -> predict) on every
sub-part of the five BASELINE configs.

* Fits: the device variogram fit of each part against the LIVE reference's
  fit of that part (tests/golden/reference_fits.json, written by
  tests/golden/make_golden_fits.py with volkrig.kriging.fit_variogram) at
  SURVEY Appendix A.5's gate |dnug| <= 1e-7 sill, |dsill| <= 1e-6 sill,
  |drange| <= 1e-4 range -- and bit for bit: the device TRF restates scipy's
  trf_bounds with numpy's/OpenBLAS's arithmetic (trf.h, npref.h, gesdd.h)
  and the svar / bin sums numpy computes (vk_npstats.cu).  The parts listed
  in CUBE_PARTS are the only ones the host restatement does not reproduce
  bit for bit (np.power(x, 3) runs through SVML pow8_ha; trf.h uses the
  correctly rounded cube), and they stay far inside the gate.
* Volumes: the device volume (device fits) against the CPU oracle's
  per-part fill driven by the reference's fitted models, all parts, at the
  fp64 gate (1e-6 of the intensity range, rint within +-1 grey level) and
  the fp32 gate (1e-3) for the fp32 configs.
"""

import numpy as np
import pytest

import fullsize as FS
from oracle import kriging_oracle as O

pytestmark = [pytest.mark.gpu]

G = FS.golden_fits()
GATE = {"nugget": 1e-7, "sill": 1e-6, "range_len": 1e-4}
# (config, part) whose host restatement differs from scipy only through x**3
CUBE_PARTS = {("C3", 2), ("C3", 14), ("C4", 25)}
_SLICES = {}


def slices(name):
    if name not in _SLICES:
        ks = FS.known_slices(name)
        assert FS.sha256(ks) == G["configs"][name]["sha256"], \
            f"{name}: regenerated phantom differs from the one the goldens were fitted on"
        _SLICES.clear()                                   # keep one config resident
        _SLICES[name] = ks
    return _SLICES[name]


def gate_ratio(dev, ref):
    sill = ref["sill"]
    return max(abs(dev.nugget - ref["nugget"]) / sill / GATE["nugget"],
               abs(dev.sill - ref["sill"]) / sill / GATE["sill"],
               abs(dev.range_len - ref["range_len"]) / ref["range_len"] / GATE["range_len"])


def device_run(torch, name, accum="fp64"):
    from paper_2303_09523_b200 import ZPartKriging
    from paper_2303_09523_b200.phantoms import CONFIGS
    cfg = CONFIGS[name]
    zk = ZPartKriging(cfg.n_known, cfg.height, cfg.width, cfg.factor, cfg.n_subparts, accum=accum)
    out, _ = zk.run(torch.from_numpy(slices(name)).cuda())
    models, _ = zk.finish()
    return cfg, zk, out, models


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_device_fits_match_reference(cuda, name):
    _, _, _, models = device_run(cuda, name)
    parts = G["configs"][name]["parts"]
    assert len(models) == len(parts)
    worst, exact, misses = 0.0, 0, []
    for p, m in zip(parts, models):
        r = gate_ratio(m, p)
        worst = max(worst, r)
        same = (m.nugget, m.sill, m.range_len) == (p["nugget"], p["sill"], p["range_len"])
        exact += same
        if not same and (name, p["part"]) not in CUBE_PARTS:
            misses.append((p["part"], r))
    print(f"\n{name}: {exact}/{len(parts)} parts bit-identical to the reference fit, "
          f"worst gate ratio {worst:.3g}")
    assert worst <= 1.0
    assert not misses, f"parts not bit-identical to the reference fit: {misses}"


@pytest.mark.parametrize("name,accum", [("C1", "fp64"), ("C2", "fp64"), ("C3", "fp32"),
                                        ("C3", "fp64"), ("C4", "fp64"), ("C5", "fp32"),
                                        ("C5", "fp64")])
def test_shipped_path_volume_matches_oracle(cuda, name, accum):
    torch = cuda
    cfg, zk, out, models = device_run(torch, name, accum)
    ks = slices(name)
    rng = float(ks.max() - ks.min())
    ref_models = [(p["nugget"], p["sill"], p["range_len"]) for p in G["configs"][name]["parts"]]
    integer = cfg.quantise in ("u8", "u12")
    worst, worst_rint = 0.0, 0.0
    for s, b, e, ref in FS.oracle_parts(ks, cfg.factor, zk.ranges, ref_models):
        z0 = b * cfg.factor
        dev = out[z0:z0 + ref.shape[0]].cpu().numpy()
        assert np.array_equal(dev[::cfg.factor], ref[::cfg.factor]), f"part {s}: known planes"
        err = float(np.abs(dev.astype(np.float64) - ref).max()) / rng
        worst = max(worst, err)
        if integer:
            worst_rint = max(worst_rint, float(np.abs(np.rint(dev) - np.rint(ref)).max()))
    tol = 1e-6 if accum == "fp64" else 1e-3
    print(f"\n{name} {accum}: max |device - oracle| = {worst:.3e} of the range over "
          f"{len(ref_models)} parts" + (f", rint diff {worst_rint:.0f}" if integer else ""))
    assert worst <= tol
    if integer and accum == "fp64":
        assert worst_rint <= 1.0
