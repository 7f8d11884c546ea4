"""GPU parity of the fixed-point tensor-core prediction (accum="fixed")
against the CPU oracle, held to the fp64 gate (max-abs <= 1e-6 of the known
intensity range, known planes bit-exact, integer grey levels within +-1).

The path quantises known values to 24-bit fixed point over the volume's range
and the kriging weights to 32-bit fixed point, then accumulates the byte
products exactly on the int8 tensor cores (vk_predict_fixed.cu).  Its error
budget is ~2e-7 of the range; these tests check it on every gap size G = 1..8,
odd widths / heights (partial tiles, border rows and columns), both drifts,
offset data (|values| >> range), the variance output and full-size C2/C4."""

import numpy as np
import pytest

from oracle import kriging_oracle as O

pytestmark = pytest.mark.gpu

TOL64 = 1e-6


def _rng(a):
    return float(np.max(a) - np.min(a))


def _run(torch, ks, cfg, accum, models=None, fit=True, variance=False, drift="linear"):
    from paper_2303_09523_b200 import ZPartKriging
    zk = ZPartKriging(cfg.n_known, cfg.height, cfg.width, cfg.factor, cfg.n_subparts,
                      accum=accum, fit=fit, drift=drift)
    out, var = zk.run(torch.from_numpy(ks).cuda(), return_variance=variance, models=models)
    m, _ = zk.finish()
    return out.cpu().numpy(), (var.cpu().numpy() if var is not None else None), m, zk


@pytest.mark.parametrize("f", [2, 3, 4, 5, 6, 7, 8, 9])
def test_fixed_vs_oracle_all_gap_sizes(cuda, f):
    torch = cuda
    from paper_2303_09523_b200.phantoms import known_slices, small_config
    cfg = small_config("head", 37, 200, 9, f, n_subparts=2, seed=f)
    ks = known_slices(cfg)
    ref, rvar, rmodels = O.reconstruct_zparts(ks, cfg.factor, cfg.n_subparts, return_variance=True)
    got, var, _, zk = _run(torch, ks, cfg, "fixed", models=rmodels, fit=False, variance=True)
    # the z-extent schedule 4 -> 8 -> 16 (kriging.py:444-457) brackets every
    # missing plane by exactly its two neighbours only for f in {2, 4, 8}; the
    # other factors take the generic fp64 path (still checked here)
    assert zk.plan.info["fast_path"] == (1 if f in (2, 4, 8) else 0)
    assert np.array_equal(got[::cfg.factor], ks)
    err = np.abs(got.astype(np.float64) - ref).max() / _rng(ks)
    assert err <= TOL64, err
    assert np.allclose(var, rvar, rtol=1e-7, atol=1e-9 * max(m.sill for m in rmodels))


@pytest.mark.parametrize("W,H", [(64, 33), (128, 32), (136, 70), (260, 41)])
@pytest.mark.parametrize("drift", ["linear", "constant"])
def test_fixed_matches_fp64_device(cuda, W, H, drift):
    torch = cuda
    from paper_2303_09523_b200.phantoms import known_slices, small_config
    cfg = small_config("brain", H, W, 7, 4, n_subparts=3, seed=W + H)
    ks = known_slices(cfg)
    ref, _, rmodels = O.reconstruct_zparts(ks, cfg.factor, cfg.n_subparts, drift=drift)
    a, _, _, _ = _run(torch, ks, cfg, "fp64", models=rmodels, fit=False, drift=drift)
    b, _, _, _ = _run(torch, ks, cfg, "fixed", models=rmodels, fit=False, drift=drift)
    r = _rng(ks)
    assert np.array_equal(a[::cfg.factor], b[::cfg.factor])
    assert np.abs(a.astype(np.float64) - b).max() <= TOL64 * r
    assert np.abs(b.astype(np.float64) - ref).max() <= TOL64 * r


def test_fixed_offset_data(cuda):
    """values ~ 1e4 + small range: the constant part L * sum(w) is carried
    separately, so the error stays relative to the range, not the level"""
    torch = cuda
    from paper_2303_09523_b200.phantoms import known_slices, small_config
    cfg = small_config("spine", 48, 96, 6, 5, n_subparts=2, seed=11)
    ks = (known_slices(cfg).astype(np.float64) * 0.01 + 1.0e4).astype(np.float32)
    ref, _, rmodels = O.reconstruct_zparts(ks, cfg.factor, cfg.n_subparts)
    got, _, _, _ = _run(torch, ks, cfg, "fixed", models=rmodels, fit=False)
    ulp = float(np.spacing(np.float32(np.abs(ks).max())))
    err = np.abs(got.astype(np.float64) - ref).max()
    assert err <= TOL64 * _rng(ks) + ulp, (err, ulp, _rng(ks))


def test_fixed_constant_volume(cuda):
    torch = cuda
    from paper_2303_09523_b200.phantoms import small_config
    from paper_2303_09523_b200 import VariogramModel
    cfg = small_config("head", 40, 64, 5, 3, n_subparts=1, seed=1)
    ks = np.full((cfg.n_known, cfg.height, cfg.width), 37.0, np.float32)
    got, _, _, _ = _run(torch, ks, cfg, "fixed",
                        models=[VariogramModel("exponential", 0.0, 1.0, 5.0)], fit=False)
    assert np.all(got == 37.0)


def test_fixed_fitted_pipeline_c1(cuda):
    torch = cuda
    from paper_2303_09523_b200.phantoms import CONFIGS, known_slices
    cfg = CONFIGS["C1"]
    ks = known_slices(cfg)
    got, _, models, _ = _run(torch, ks, cfg, "fixed")
    ref, _, rmodels = O.reconstruct_zparts(ks, cfg.factor, cfg.n_subparts)
    assert np.array_equal(got[::cfg.factor], ks)
    assert np.abs(np.rint(got) - np.rint(ref)).max() <= 1
    fp, _, _, _ = _run(torch, ks, cfg, "fp64")
    # same device fit -> the two predictions differ only by the fixed-point error
    assert np.abs(got.astype(np.float64) - fp).max() <= TOL64 * _rng(ks)


def test_fixed_c4_full_size_sampled(cuda):
    """Full C4 (512^2, K=256, f=8, 32 parts) with the oracle's models on three
    parts: sampled voxels against the oracle at the fp64 gate, and the whole
    volume against the device fp64 path."""
    torch = cuda
    from paper_2303_09523_b200 import VariogramModel, ZPartKriging
    from paper_2303_09523_b200.phantoms import CONFIGS, known_slices
    cfg = CONFIGS["C4"]
    ks = known_slices(cfg)
    f = cfg.factor
    kd = torch.from_numpy(ks).cuda()
    zk = ZPartKriging(cfg.n_known, cfg.height, cfg.width, f, cfg.n_subparts)
    zk.run(kd)
    dev_models, _ = zk.finish()
    ranges = O.subpart_ranges(cfg.n_known, cfg.n_subparts)
    parts = [0, 17, cfg.n_subparts - 1]
    ref_models = {}
    for s in parts:
        b, e = ranges[s]
        d, m = O.subpart_grid(ks, b, e, f)
        ref_models[s] = O.fit_variogram(O.subpart_samples(d, m))
    models = [ref_models.get(s, dev_models[s]) for s in range(cfg.n_subparts)]
    models = [VariogramModel("exponential", m.nugget, m.sill, m.range_len) for m in models]
    outs = {}
    for accum in ("fp64", "fixed"):
        z = ZPartKriging(cfg.n_known, cfg.height, cfg.width, f, cfg.n_subparts, fit=False, accum=accum)
        o, _ = z.run(kd, models=models)
        z.finish()
        outs[accum] = o
    r = _rng(ks)
    diff = (outs["fp64"].double() - outs["fixed"].double()).abs().max().item()
    assert diff <= TOL64 * r, diff / r
    vol = outs["fixed"].cpu().numpy()
    assert np.array_equal(vol[::f], ks)
    from test_gpu_fullsize import _oracle_voxels
    rng = np.random.default_rng(1)
    for s in parts:
        b, e = ranges[s]
        depth = (e - b) * f + 1
        zl = rng.integers(0, depth, 300)
        zl = zl[zl % f != 0]
        yl = np.concatenate([rng.integers(0, cfg.height, len(zl) - 4), [0, 1, cfg.height - 2, cfg.height - 1]])
        xl = np.concatenate([rng.integers(0, cfg.width, len(zl) - 4), [0, cfg.width - 1, 1, cfg.width - 2]])
        zyx = np.stack([zl, yl[:len(zl)], xl[:len(zl)]], 1)
        exp = _oracle_voxels(ks, b, e, f, ref_models[s], "linear", zyx)
        got = vol[b * f + zyx[:, 0], zyx[:, 1], zyx[:, 2]].astype(np.float64)
        assert np.abs(got - exp).max() <= TOL64 * r
        assert np.abs(np.rint(got) - np.rint(exp)).max() <= 1


def test_fixed_linear_field_full_size_c2(cuda):
    torch = cuda
    from paper_2303_09523_b200 import ZPartKriging
    from paper_2303_09523_b200.phantoms import CONFIGS
    cfg = CONFIGS["C2"]
    K, H, W, f = cfg.n_known, cfg.height, cfg.width, cfg.factor
    z = (np.arange(K) * f).astype(np.float32)[:, None, None]
    y = np.arange(H, dtype=np.float32)[None, :, None]
    x = np.arange(W, dtype=np.float32)[None, None, :]
    ks = (0.25 * x + 0.5 * y + 0.125 * z + 3.0).astype(np.float32)
    zk = ZPartKriging(K, H, W, f, cfg.n_subparts, accum="fixed")
    out, _ = zk.run(torch.from_numpy(ks).cuda())
    zk.finish()
    T = out.shape[0]
    zz = torch.arange(T, device="cuda", dtype=torch.float64)[:, None, None]
    yy = torch.arange(H, device="cuda", dtype=torch.float64)[None, :, None]
    xx = torch.arange(W, device="cuda", dtype=torch.float64)[None, None, :]
    err = (out.double() - (0.25 * xx + 0.5 * yy + 0.125 * zz + 3.0)).abs().max().item()
    assert err <= TOL64 * float(ks.max() - ks.min()), err
