"""Generate golden vectors from the LIVE reference (volkrig, read-only at
/root/reference/pkg/src).  Run in the build container only:

    python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs on seeded inputs
are committed here as small fixtures; tests/ compare both the CPU oracle and
the CUDA path against them.  Inputs are regenerated from the seeds recorded
in the fixtures (numpy default_rng and paper_2303_09523_b200.phantoms).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import scipy

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)

from volkrig import errors as E          # noqa: E402
from volkrig import kriging as K         # noqa: E402
from volkrig import model as M           # noqa: E402

from paper_2303_09523_b200.phantoms import known_slices, small_config  # noqa: E402
sys.path.insert(0, HERE)
from golden_inputs import smooth_grid  # noqa: E402


def _env():
    import numpy.__config__ as npc
    blas = npc.CONFIG.get("Build Dependencies", {}).get("blas", {})
    return {"numpy": np.__version__, "scipy": scipy.__version__,
            "blas": f"{blas.get('name')} {blas.get('version')}"}


FILL_CASES = [
    # (name, seed, T, H, W, known_z, kind, nugget, sill, range, drift, variance)
    ("f2_lin", 1, 9, 21, 28, range(0, 9, 2), "exponential", 0.5, 400.0, 15.0, "linear", True),
    ("f3_lin", 2, 13, 20, 24, range(0, 13, 3), "exponential", 0.0, 300.0, 40.0, "linear", True),
    ("f4_lin", 3, 13, 24, 32, range(0, 13, 4), "exponential", 2.0, 500.0, 25.0, "linear", True),
    ("f4_const", 3, 13, 24, 32, range(0, 13, 4), "exponential", 2.0, 500.0, 25.0, "constant", True),
    ("f5_lin", 4, 16, 18, 20, range(0, 16, 5), "exponential", 1.0, 250.0, 30.0, "linear", False),
    ("f8_lin", 5, 17, 16, 24, range(0, 17, 8), "exponential", 0.1, 800.0, 60.0, "linear", True),
    ("f16_lin", 6, 33, 12, 16, range(0, 33, 16), "exponential", 0.0, 200.0, 20.0, "linear", False),
    ("irregular", 7, 15, 17, 19, (1, 2, 6, 9, 14), "exponential", 0.3, 350.0, 12.0, "linear", True),
    ("tiny_w", 8, 7, 9, 3, range(0, 7, 2), "exponential", 0.0, 100.0, 5.0, "linear", True),
    ("tiny_hw", 9, 5, 2, 3, range(0, 5, 2), "exponential", 0.0, 100.0, 5.0, "constant", False),
    ("gauss", 10, 9, 16, 20, range(0, 9, 4), "gaussian", 1.0, 300.0, 8.0, "linear", False),
    ("spher", 11, 9, 16, 20, range(0, 9, 4), "spherical", 1.0, 300.0, 10.0, "linear", True),
    ("white", 12, 9, 12, 16, range(0, 9, 2), "exponential", 0.0, 0.0, 1.0, "linear", False),
    ("float_vals", 13, 9, 20, 32, range(0, 9, 4), "exponential", 1e-4, 0.02, 30.0, "linear", True),
]


def make_fill(out):
    meta = []
    for (name, seed, T, H, W, kz, kind, nug, sill, rng, drift, var) in FILL_CASES:
        data, mask = smooth_grid(seed, T, H, W, kz, quant=name != "float_vals")
        if name == "float_vals":
            data = np.where(mask, np.nan, data / 220.0).astype(np.float32)
        g = M.VolumeGrid(data, mask)
        mdl = K.VariogramModel(kind, nug, sill, rng)
        res = K.fill_missing(g, mdl, drift, return_variance=var)
        grid, v = (res if var else (res, None))
        out[f"fill_{name}_out"] = grid.data
        if var:
            out[f"fill_{name}_var"] = v
        meta.append({"name": name, "seed": seed, "shape": [T, H, W], "known_z": list(kz),
                     "kind": kind, "model": [nug, sill, rng], "drift": drift,
                     "variance": var, "quant": name != "float_vals"})
    return meta


def make_systems(out):
    """Weights / variance of the stencil families of the plane fill."""
    meta = []
    models = [("exponential", 0.0, 500.0, 30.0), ("exponential", 5.0, 500.0, 200.0),
              ("exponential", 0.0, 0.0, 1.0), ("spherical", 1.0, 300.0, 12.0)]
    fams = []
    for f in (2, 4, 8):
        for j in range(1, f):
            fams.append((-j, f - j))
    fams += [(-7,), (8,), (-2, 1, 4)]
    xk = {"I": range(-1, 3), "L": range(0, 3), "R1": range(-1, 2), "R2": range(-1, 1)}
    i = 0
    for dz in fams:
        for kx in ("I", "L", "R2"):
            for ky in ("I", "R1"):
                rel = np.array([(ox, oy, oz) for oz in dz for oy in xk[ky] for ox in xk[kx]],
                               dtype=np.int64)
                for mi, (kind, nug, sill, rng) in enumerate(models):
                    for drift in ("linear", "constant"):
                        mdl = K.VariogramModel(kind, nug, sill, rng)
                        sys_ = K.solve_ked(K.build_system(rel, np.zeros(len(rel)), (0, 0, 0),
                                                          mdl, drift))
                        out[f"sys_{i}_rel"] = rel
                        out[f"sys_{i}_w"] = sys_.weights
                        out[f"sys_{i}_lam"] = sys_.lagrange
                        meta.append({"id": i, "model": [kind, nug, sill, rng], "drift": drift,
                                     "variance": sys_.variance})
                        i += 1
    return meta


def make_fit(out):
    meta = []
    r = np.random.default_rng(21)
    cases = []
    for m in (40, 300, 447, 448, 3000):                  # triu path and RNG path
        c = r.integers(0, 40, size=(m, 3)).astype(float)
        v = np.sin(c[:, 0] / 7) * 10 + c[:, 2] + r.normal(size=m)
        cases.append((f"rand_{m}", c, v))
    for fam, seed in (("head", 31), ("spine", 32), ("brain", 33)):
        cfg = small_config(fam, 40, 48, 5, 4, n_subparts=1, seed=seed)
        ks = known_slices(cfg)
        T = cfg.depth
        data = np.full((T,) + ks.shape[1:], np.nan, np.float32)
        data[::cfg.factor] = ks
        mask = np.isnan(data)
        kz, ky, kx = np.nonzero(~mask)
        coords = np.column_stack([kx, ky, kz]).astype(float)
        cases.append((f"phantom_{fam}", coords, data[kz, ky, kx].astype(float)))
    for name, c, v in cases:
        for kind in ("exponential", "gaussian", "spherical"):
            mdl = K.fit_variogram((c, v), kind=kind)
            key = f"fit_{name}_{kind}"
            out[key + "_coords"] = c
            out[key + "_values"] = v
            meta.append({"key": key, "kind": kind,
                         "model": [mdl.nugget, mdl.sill, mdl.range_len]})
    # pair draws (numpy RNG, seed 0) for the device PCG64 kernel
    import hashlib
    pairs = {}
    for m in (500, 81_920, 327_680, 2_359_296, 9_437_184):
        g = np.random.default_rng(0)
        ii = g.integers(0, m, size=100_000).astype(np.int32)
        jj = g.integers(0, m, size=100_000).astype(np.int32)
        out[f"pairs_{m}_ii_head"] = ii[:1000]
        out[f"pairs_{m}_jj_head"] = jj[:1000]
        pairs[str(m)] = {"ii_sha256": hashlib.sha256(ii.tobytes()).hexdigest(),
                         "jj_sha256": hashlib.sha256(jj.tobytes()).hexdigest()}
    meta.append({"key": "pairs", "draws": pairs})
    return meta


def make_pipeline(out):
    """Per-Z-part fit_variogram + fill_missing on phantoms."""
    meta = []
    for name, cfg in (("head_small", small_config("head", 48, 64, 9, 2, 2, seed=3)),
                      ("spine_small", small_config("spine", 40, 64, 9, 4, 2, seed=7))):
        ks = known_slices(cfg)
        K_ = ks.shape[0]
        q = K_ // cfg.n_subparts
        vol = np.empty((cfg.depth,) + ks.shape[1:], np.float32)
        models = []
        for s in range(cfg.n_subparts):
            b, e = s * q, ((s + 1) * q if s < cfg.n_subparts - 1 else K_ - 1)
            depth = (e - b) * cfg.factor + 1
            data = np.full((depth,) + ks.shape[1:], np.nan, np.float32)
            data[::cfg.factor] = ks[b:e + 1]
            g = M.VolumeGrid(data)
            kz, ky, kx = np.nonzero(~g.missing_mask)
            coords = np.column_stack([kx, ky, kz]).astype(float)
            mdl = K.fit_variogram((coords, data[kz, ky, kx].astype(float)))
            filled = K.fill_missing(g, mdl, "linear")
            vol[b * cfg.factor:b * cfg.factor + depth] = filled.data
            models.append([mdl.nugget, mdl.sill, mdl.range_len])
        out[f"pipe_{name}_known"] = ks
        out[f"pipe_{name}_out"] = vol
        meta.append({"name": name, "factor": cfg.factor, "n_subparts": cfg.n_subparts,
                     "models": models})
    return meta


def make_kats():
    """SPEC.md examples that hold against the reference."""
    k = {}
    s1 = K.solve_ked(K.build_system([(0, 0, 1)], [3.0], (0, 0, 0),
                                    K.VariogramModel("exponential", 0, 1, 5), "constant"))
    k["single_neighbour_w"] = float(s1.weights[0])
    pts = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0)]
    s4 = K.solve_ked(K.build_system(pts, [2.0] * 4, (0, 0, 0),
                                    K.VariogramModel("exponential", 0, 1, 5), "constant"))
    k["four_symmetric_w"] = [float(w) for w in s4.weights]
    # linear field reproduced exactly with linear drift
    T, H, W = 9, 12, 14
    z, y, x = np.meshgrid(np.arange(T), np.arange(H), np.arange(W), indexing="ij")
    field = (2 * x + 3 * y + z).astype(np.float32)
    data = field.copy()
    data[1::2] = np.nan
    g = K.fill_missing(M.VolumeGrid(data), K.VariogramModel("exponential", 0, 1, 5), "linear")
    k["linear_field_maxerr"] = float(np.abs(g.data - field)[1::2].max())
    # constant planes with g = 4
    data = np.full((11, 8, 9), np.nan, np.float32)
    data[::5] = 0.75
    g = K.fill_missing(M.VolumeGrid(data), K.VariogramModel("exponential", 0, 1, 5), "linear")
    k["constant_planes_maxerr"] = float(np.abs(g.data - 0.75).max())
    # z ramp with linear drift
    data = np.full((9, 8, 9), np.nan, np.float32)
    for i in range(0, 9, 4):
        data[i] = i / 8.0
    g = K.fill_missing(M.VolumeGrid(data), K.VariogramModel("exponential", 0, 1, 5), "linear")
    ramp = (np.arange(9) / 8.0)[:, None, None]
    k["z_ramp_maxerr"] = float(np.abs(g.data - ramp).max())
    return k


def make_errors():
    """Exception classes the reference raises on boundary inputs."""
    cases = {}

    def name(fn):
        try:
            fn()
            return None
        except Exception as exc:   # noqa: BLE001
            return type(exc).__name__

    cases["insufficient_samples"] = name(lambda: K.fit_variogram(
        (np.zeros((7, 3)), np.arange(7.0))))
    cases["degenerate_lags"] = name(lambda: K.fit_variogram(
        (np.zeros((20, 3)), np.arange(20.0))))
    d = np.full((3, 4, 4), np.nan, np.float32)
    cases["no_known"] = name(lambda: K.fill_missing(
        M.VolumeGrid(d), K.VariogramModel("exponential", 0, 1, 1)))
    d2 = np.zeros((3, 4, 4), np.float32)
    m2 = np.zeros((3, 4, 4), bool)
    m2[1] = True
    cases["mask_out_of_sync"] = name(lambda: K.fill_missing(
        M.VolumeGrid(d2, m2), K.VariogramModel("exponential", 0, 1, 1)))
    d3 = np.full((3, 4, 4), np.nan, np.float32)
    d3[0] = 1.0
    d3[2] = np.inf
    cases["known_not_finite"] = name(lambda: K.fill_missing(
        M.VolumeGrid(d3, np.isnan(d3) | False), K.VariogramModel("exponential", 0, 1, 1)))
    cases["bad_kind"] = name(lambda: K.VariogramModel("linear", 0, 1, 1))
    cases["bad_model"] = name(lambda: K.VariogramModel("exponential", 2, 1, 1))
    cases["unknown_drift"] = name(lambda: K.fill_missing(
        M.VolumeGrid(np.where(np.arange(27).reshape(3, 3, 3) // 9 == 1, np.nan,
                              1.0).astype(np.float32)),
        K.VariogramModel("exponential", 0, 1, 1), drift="quadratic"))
    # dense grid: unchanged, no error
    cases["dense_grid"] = name(lambda: K.fill_missing(
        M.VolumeGrid(np.ones((2, 3, 3), np.float32)), K.VariogramModel("exponential", 0, 1, 1)))
    assert issubclass(E.SingularSystem, E.VolkrigError)
    return cases


def main():
    out = {}
    meta = {"env": _env(), "fill": make_fill(out), "systems": make_systems(out),
            "fit": make_fit(out), "pipeline": make_pipeline(out), "kats": make_kats(),
            "errors": make_errors()}
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", len(out), "arrays;", meta["env"])


if __name__ == "__main__":
    main()
