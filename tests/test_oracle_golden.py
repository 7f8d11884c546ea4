"""CPU: the oracle (numpy restatement) against the golden vectors the live
reference produced (tests/golden/make_golden.py), and against the reference
itself when it is importable (build container only)."""

import json
import os
import sys

import numpy as np
import pytest

from oracle import kriging_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "reference_golden.npz"))
META = json.load(open(os.path.join(HERE, "golden", "reference_golden.json")))
sys.path.insert(0, os.path.join(HERE, "golden"))
from golden_inputs import smooth_grid  # noqa: E402  (input regeneration only)

REF = "/root/reference/pkg/src"


def fill_inputs(c):
    data, mask = smooth_grid(c["seed"], *c["shape"], c["known_z"], quant=c["quant"])
    if not c["quant"]:
        data = np.where(mask, np.nan, data / 220.0).astype(np.float32)
    return data, mask


@pytest.mark.parametrize("case", META["fill"], ids=lambda c: c["name"])
def test_fill_matches_reference(case):
    data, mask = fill_inputs(case)
    out, var = O.fill_missing(data, mask, O.Model(case["kind"], *case["model"]),
                              case["drift"], case["variance"])
    gold = GOLD[f"fill_{case['name']}_out"]
    assert np.array_equal(out[~mask], data[~mask])                 # known: bit-exact
    assert np.allclose(out, gold, rtol=0, atol=1e-9 * np.nanmax(np.abs(gold)))
    if case["variance"]:
        assert np.allclose(var, GOLD[f"fill_{case['name']}_var"], rtol=1e-9, atol=1e-12)


def test_systems_match_reference():
    for m in META["systems"][::7]:
        rel = GOLD[f"sys_{m['id']}_rel"]
        kind, nug, sill, rng = m["model"]
        A, b, n, Q, q0 = O.assemble(rel, O.Model(kind, nug, sill, rng), m["drift"])
        w, lam, var, _ = O.solve(A, b, n, Q, q0)
        assert np.allclose(w, GOLD[f"sys_{m['id']}_w"], rtol=1e-9, atol=1e-12)
        assert abs(var - m["variance"]) <= 1e-9 * max(1.0, abs(m["variance"]))


def test_fit_matches_reference():
    for m in META["fit"]:
        if m["key"] == "pairs":
            continue
        c = GOLD[m["key"] + "_coords"]
        v = GOLD[m["key"] + "_values"]
        got = O.fit_variogram((c, v), kind=m["kind"])
        nug, sill, rng = m["model"]
        assert abs(got.nugget - nug) <= 1e-9 * max(sill, 1e-300) + 1e-12
        assert abs(got.sill - sill) <= 1e-9 * max(sill, 1e-300)
        assert abs(got.range_len - rng) <= 1e-7 * rng


def test_pair_draws_match_numpy():
    import hashlib
    draws = [m for m in META["fit"] if m["key"] == "pairs"][0]["draws"]
    for m, h in draws.items():
        m = int(m)
        ii, jj = O.pair_indices(m, 100_000, 0)
        if m * (m - 1) // 2 <= 100_000:
            continue
        # oracle drops i == j pairs; recover the raw draws through numpy
        g = np.random.default_rng(0)
        ri = g.integers(0, m, size=100_000).astype(np.int32)
        rj = g.integers(0, m, size=100_000).astype(np.int32)
        assert hashlib.sha256(ri.tobytes()).hexdigest() == h["ii_sha256"]
        assert hashlib.sha256(rj.tobytes()).hexdigest() == h["jj_sha256"]
        keep = ri != rj
        assert np.array_equal(ii, ri[keep]) and np.array_equal(jj, rj[keep])


@pytest.mark.parametrize("case", META["pipeline"], ids=lambda c: c["name"])
def test_pipeline_matches_reference(case):
    ks = GOLD[f"pipe_{case['name']}_known"]
    vol, _, models = O.reconstruct_zparts(ks, case["factor"], case["n_subparts"])
    gold = GOLD[f"pipe_{case['name']}_out"]
    rng = float(ks.max() - ks.min())
    assert np.abs(vol.astype(np.float64) - gold).max() <= 1e-6 * rng
    for m, r in zip(models, case["models"]):
        assert abs(m.sill - r[1]) <= 1e-7 * r[1]


def test_kats():
    k = META["kats"]
    assert k["single_neighbour_w"] == 1.0
    assert np.allclose(k["four_symmetric_w"], 0.25, atol=1e-12)
    for key in ("linear_field_maxerr", "constant_planes_maxerr", "z_ramp_maxerr"):
        assert k[key] <= 1e-5
    # the oracle reproduces the same examples
    w, _ = O.stencil_weights(np.array([[0, 0, 1]]), O.Model("exponential", 0, 1, 5), "constant")
    assert w[0] == 1.0
    T, H, W = 9, 12, 14
    z, y, x = np.meshgrid(np.arange(T), np.arange(H), np.arange(W), indexing="ij")
    field = (2 * x + 3 * y + z).astype(np.float32)
    data = field.copy()
    data[1::2] = np.nan
    out, _ = O.fill_missing(data, np.isnan(data), O.Model("exponential", 0, 1, 5), "linear")
    assert np.abs(out - field).max() <= 1e-5


def test_error_contract():
    e = META["errors"]
    assert e["insufficient_samples"] == "InsufficientSamples"
    assert e["degenerate_lags"] == "DegenerateLags"
    assert e["no_known"] == "NoKnownNeighbors"
    for k in ("mask_out_of_sync", "known_not_finite", "bad_kind", "bad_model", "unknown_drift"):
        assert e[k] == "ValueError"
    with pytest.raises(O.InsufficientSamples):
        O.fit_variogram((np.zeros((7, 3)), np.arange(7.0)))
    with pytest.raises(O.DegenerateLags):
        O.fit_variogram((np.zeros((20, 3)), np.arange(20.0)))


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_oracle_equals_live_reference():
    sys.path.insert(0, REF)
    from volkrig import kriging as K
    from volkrig import model as M
    r = np.random.default_rng(99)
    for f in (2, 3, 4):
        T = 3 * f + 1
        data, mask = smooth_grid(int(r.integers(1000)), T, 14, 17, range(0, T, f))
        mdl = (0.3, 250.0, 20.0)
        exp = K.fill_missing(M.VolumeGrid(data, mask), K.VariogramModel("exponential", *mdl))
        got, _ = O.fill_missing(data, mask, O.Model("exponential", *mdl))
        assert np.array_equal(got, exp.data)
        kz, ky, kx = np.nonzero(~mask)
        c = np.column_stack([kx, ky, kz]).astype(float)
        v = data[kz, ky, kx].astype(float)
        a = K.fit_variogram((c, v))
        b = O.fit_variogram((c, v))
        assert (a.nugget, a.sill, a.range_len) == (b.nugget, b.sill, b.range_len)


# --------------------------------------------------------------------------
# generic per-voxel path (non-plane masks), tests/golden/make_golden_generic.py
# --------------------------------------------------------------------------

def _generic_golden():
    d = np.load(os.path.join(HERE, "golden", "reference_generic.npz"))
    with open(os.path.join(HERE, "golden", "reference_generic.json")) as f:
        meta = json.load(f)
    return d, meta


def test_oracle_generic_path_matches_reference_goldens():
    d, meta = _generic_golden()
    assert len(meta["cases"]) >= 7
    for c in meta["cases"]:
        n = c["name"]
        kind, nug, sill, rng = c["model"]
        out, var = O.fill_missing(d[f"{n}/data"], d[f"{n}/mask"], O.Model(kind, nug, sill, rng),
                                  c["drift"], True)
        assert O.plane_flags(d[f"{n}/mask"]) is None
        np.testing.assert_array_equal(out, d[f"{n}/out"], err_msg=n)
        np.testing.assert_allclose(var, d[f"{n}/var"], rtol=1e-12, atol=1e-12 * sill, err_msg=n)


def test_oracle_generic_no_neighbors():
    _, meta = _generic_golden()
    nn = meta["no_neighbors"]
    data = np.full(nn["shape"], np.nan, np.float32)
    data[0, 0, nn["known_x"]] = 5.0
    with pytest.raises(O.NoKnownNeighbors, match=r"\(8, 0, 0\)"):
        O.fill_missing(data, np.isnan(data), O.Model("exponential", 0.0, 1.0, 3.0))


def test_oracle_generic_window_schedule():
    """kriging.py:39, 414-424: bracketing decides the z extent; at z extent
    16 the first window with any known voxel is taken."""
    mask = np.ones((20, 9, 9), bool)
    mask[3] = False                                   # known plane below z=10 only
    i, coords = O.choose_window(mask, 4, 4, 10)
    assert O.WINDOW_SCHEDULE[i] == (4, 16) and set(coords[:, 2]) == {3}
    mask[12] = False                                  # above only at z extent 8 (planes 7..14)
    i, coords = O.choose_window(mask, 4, 4, 10)
    assert O.WINDOW_SCHEDULE[i] == (4, 16) and set(coords[:, 2]) == {3, 12}
    mask[8] = False                                   # bracketed at z extent 8
    i, coords = O.choose_window(mask, 4, 4, 10)
    assert O.WINDOW_SCHEDULE[i] == (4, 8) and set(coords[:, 2]) == {8, 12}
