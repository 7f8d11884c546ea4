"""CPU: header-only device code compiled for the host (test shim) against
numpy / scipy / the oracle: SeedSequence+PCG64 state, Lemire draws, the TRF
fit, and the plane-window / stencil geometry."""

import ctypes as C
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import kriging_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
META = json.load(open(os.path.join(HERE, "golden", "reference_golden.json")))
I32 = C.POINTER(C.c_int32)
D = C.POINTER(C.c_double)


@pytest.fixture(scope="module")
def shim():
    import native_build
    return native_build.build_shim()


def test_seedsequence_pcg64_state(shim):
    out = (C.c_uint64 * 4)()
    for seed in (0, 1, 7, 12345, 2 ** 40 + 3):
        shim.vkh_pcg_state(C.c_uint64(seed), out)
        st = np.random.PCG64(seed).state["state"]
        assert (out[0] << 64 | out[1]) == st["state"]
        assert (out[2] << 64 | out[3]) == st["inc"]


def test_lemire_draws_match_numpy(shim):
    draws = [m for m in META["fit"] if m["key"] == "pairs"][0]["draws"]
    for m, h in draws.items():
        m = int(m)
        buf = np.zeros(200_000, np.int64)
        shim.vkh_draws(C.c_uint64(0), C.c_uint32(m), C.c_int64(100_000),
                       buf.ctypes.data_as(C.POINTER(C.c_int64)))
        ii, jj = buf[:100_000].astype(np.int32), buf[100_000:].astype(np.int32)
        assert hashlib.sha256(ii.tobytes()).hexdigest() == h["ii_sha256"], m
        assert hashlib.sha256(jj.tobytes()).hexdigest() == h["jj_sha256"], m


def _trf(shim, b, kind):
    nz = b.counts > 0
    h = np.ascontiguousarray((0.5 * (b.edges[:-1] + b.edges[1:]))[nz])
    g = np.ascontiguousarray(b.sums[nz] / b.counts[nz])
    w = np.ascontiguousarray(np.sqrt(b.counts[nz].astype(float)))
    x0 = np.array([0.0, b.svar, b.hmax / 3])
    lb = np.array([0.0, 0.0, 1e-6])
    ub = np.array([2 * b.svar + 1e-12, 4 * b.svar + 1e-12, 10 * b.hmax])
    x = np.zeros(3)
    info = np.zeros(3, np.int32)
    shim.vkh_trf(O.KINDS.index(kind), len(h), h.ctypes.data_as(D), g.ctypes.data_as(D),
                 w.ctypes.data_as(D), x0.ctypes.data_as(D), lb.ctypes.data_as(D),
                 ub.ctypes.data_as(D), x.ctypes.data_as(D), info.ctypes.data_as(I32))
    nug = max(x[0], 0.0)
    return O.Model(kind, nug, nug + max(x[1], 0.0), max(x[2], 1e-6)), info


def test_trf_restatement_vs_scipy(shim):
    """trf.h restates scipy's trf_bounds with numpy's arithmetic: the fit lands
    on scipy's end point (SURVEY Appendix A.5 gate) and the fill agrees at the
    fp64 gate (bit-identity on the BASELINE parts: tests/test_fit_parity.py)."""
    from paper_2303_09523_b200.phantoms import known_slices, small_config
    for fam, seed in (("head", 3), ("spine", 7), ("brain", 5)):
        cfg = small_config(fam, 48, 64, 9, 4, n_subparts=2, seed=seed)
        ks = known_slices(cfg)
        for (b, e) in O.subpart_ranges(cfg.n_known, cfg.n_subparts):
            d, m = O.subpart_grid(ks, b, e, cfg.factor)
            c, v = O.subpart_samples(d, m)
            bins = O.empirical_bins(c, v)
            got, info = _trf(shim, bins, "exponential")
            ref = O.fit_bins(bins, "exponential")
            assert info[0] > 0
            assert abs(got.sill - ref.sill) <= 1e-6 * ref.sill
            assert abs(got.nugget - ref.nugget) <= 1e-7 * ref.sill
            assert abs(got.range_len - ref.range_len) <= 1e-4 * ref.range_len
            o1, _ = O.fill_missing(d, m, ref)
            o2, _ = O.fill_missing(d, m, got)
            assert np.abs(o1.astype(float) - o2).max() <= 1e-6 * float(ks.max() - ks.min())


def _geometry(shim, H, W, kz, S=1, drift=0):
    T = int(kz[-1]) + 1 if not isinstance(kz, tuple) else kz[1]
    kz = np.ascontiguousarray(kz[0] if isinstance(kz, tuple) else kz, np.int32)
    info = np.zeros(6, np.int32)
    n = T * 8
    mz = np.zeros(T, np.int32)
    mp = np.zeros(T * 8, np.int32)
    po = np.zeros(n * 8, np.int32)
    pn = np.zeros(n, np.int32)
    st = np.zeros(n * 64 * 5, np.int32)
    err = C.create_string_buffer(256)
    rc = shim.vkh_geometry(H, W, T, kz.ctypes.data_as(I32), len(kz), S, drift,
                           info.ctypes.data_as(I32), mz.ctypes.data_as(I32), mp.ctypes.data_as(I32),
                           po.ctypes.data_as(I32), pn.ctypes.data_as(I32), st.ctypes.data_as(I32),
                           err, 256)
    return rc, err.value.decode(), info, mz, mp.reshape(-1, 8), po.reshape(-1, 8), pn, st.reshape(-1, 5)


@pytest.mark.parametrize("layout", [
    (np.arange(0, 9, 2), 9), (np.arange(0, 13, 3), 13), (np.arange(0, 13, 4), 13),
    (np.arange(0, 16, 5), 16), (np.arange(0, 17, 8), 17), (np.arange(0, 33, 16), 33),
    (np.array([1, 2, 6, 9, 14]), 15), (np.array([3, 4, 5, 10]), 12)])
def test_plane_windows_match_oracle(shim, layout):
    kz, T = layout
    rc, err, info, mz, mp, po, pn, st = _geometry(shim, 10, 12, (kz, T))
    assert rc == 0, err
    n_miss = info[0]
    missing = [z for z in range(T) if z not in set(kz.tolist())]
    assert list(mz[:n_miss]) == missing
    for i, z in enumerate(missing):
        exp = O.plane_window(z, kz, T)
        got = [kz[k] for k in mp[i] if k >= 0]
        assert list(got) == list(exp)


def test_drift_columns_match_lstsq_rule(shim):
    for kz, T, drift in ((np.arange(0, 9, 4), 9, 0), (np.arange(0, 33, 16), 33, 0),
                         (np.arange(0, 9, 2), 9, 1)):
        rc, err, info, mz, mp, po, pn, st = _geometry(shim, 9, 11, (kz, T), drift=drift)
        assert rc == 0
        for (pat, ky, kx, n, cols) in st[:info[2]]:
            offs = [o for o in po[pat][:pn[pat]]]
            yr = range(ky // 3 - 1, ky % 3 + 1)
            xr = range(kx // 3 - 1, kx % 3 + 1)
            rel = np.array([(ox, oy, oz) for oz in offs for oy in yr for ox in xr], float)
            assert len(rel) == n
            kept = O.independent_drift(O.drift_columns(rel, ["linear", "constant"][drift]))
            assert cols == sum(1 << c for c in kept)


def test_fast_path_eligibility(shim):
    rc, _, info, *_ = _geometry(shim, 64, 128, np.arange(0, 57, 8), S=2)
    assert rc == 0 and info[3] == 1 and info[4] == 7
    rc, _, info, *_ = _geometry(shim, 64, 130, np.arange(0, 57, 8), S=2)
    assert rc == 0 and info[3] == 0                      # W % 4 != 0 -> generic
    rc, _, info, *_ = _geometry(shim, 64, 128, np.arange(0, 13, 3))
    assert rc == 0 and info[3] == 0                      # f = 3 reads 3 planes


def test_geometry_errors(shim):
    rc, err, *_ = _geometry(shim, 8, 8, (np.array([0, 40]), 41))
    assert rc == 1 and err.startswith("NoKnownNeighbors")
    rc, err, *_ = _geometry(shim, 8, 8, (np.array([3, 2]), 5))
    assert rc == 1 and err.startswith("Invalid")


@pytest.mark.parametrize("H,W,f,K,S", [(24, 40, 8, 3, 1), (20, 36, 4, 9, 2), (16, 16, 2, 7, 3)])
@pytest.mark.parametrize("drift", [0, 1])
def test_orbit_derived_systems(shim, H, W, f, K, S, drift):
    """Only one system per z-mirror / x<->y-transpose orbit is solved
    (vk_geometry.cpp canonical_systems); every derived system, rebuilt from
    its source's oracle solution by reversing planes / transposing taps, must
    equal the oracle's direct solve of its own stencil (kriging.py:159-245),
    and each part lists its solved systems first."""
    kz = np.arange(K, dtype=np.int32) * f
    T = int(kz[-1]) + 1
    nmax = T * 8 * 64
    n_out = np.zeros(2, np.int32)
    sys_ = np.zeros(nmax * 4, np.int32)
    src = np.zeros(nmax, np.int32)
    fl = np.zeros(nmax, np.int32)
    canon = np.zeros(S, np.int32)
    po = np.zeros(T * 8 * 8, np.int32)
    assert shim.vkh_orbits(H, W, T, kz.ctypes.data_as(I32), K, S, drift, n_out.ctypes.data_as(I32),
                           sys_.ctypes.data_as(I32), src.ctypes.data_as(I32), fl.ctypes.data_as(I32),
                           canon.ctypes.data_as(I32), po.ctypes.data_as(I32)) == 0
    n, nd = int(n_out[0]), int(n_out[1])
    sys_ = sys_[:n * 4].reshape(n, 4)
    src, fl = src[:n], fl[:n]
    po = po.reshape(-1, 8)
    assert nd == int((src >= 0).sum()) and nd > 0
    if f == 8 and S == 1:
        assert n == 112 and n - nd == 40            # 7 patterns x 16 kinds -> 4 x 10
    m = O.Model("exponential", 2.0, 700.0, 9.0)
    dr = "linear" if drift == 1 else "constant"
    solved = {}

    def solve(i):
        if i not in solved:
            _, p, ky, kx = sys_[i]
            offs = [o for o in po[p] if o != 99]
            rel, slots = [], []
            for pl, dz in enumerate(offs):
                for oy in range(ky // 3 - 1, ky % 3 + 1):
                    for ox in range(kx // 3 - 1, kx % 3 + 1):
                        rel.append((ox, oy, dz))
                        slots.append(pl * 16 + (oy + 1) * 4 + (ox + 1))
            w, v = O.stencil_weights(np.array(rel, float), m, dr)
            pad = np.zeros(128)
            pad[slots] = w
            solved[i] = (pad, v, len(offs))
        return solved[i]

    begin = 0
    for s in range(S):
        end = begin + int((sys_[:, 0] == s).sum())
        assert np.all(src[begin:canon[s]] < 0) and np.all(src[canon[s]:end] >= 0)
        begin = end
    for i in np.nonzero(src >= 0)[0]:
        j = int(src[i])
        assert src[j] < 0 and sys_[j, 0] == sys_[i, 0]
        wj, vj, npl = solve(j)
        wi, vi, _ = solve(int(i))
        assert fl[i] >> 8 == npl
        d = wj.reshape(8, 4, 4)
        if fl[i] & 1:
            d = np.concatenate([d[:npl][::-1], d[npl:]])
        if fl[i] & 2:
            d = d.transpose(0, 2, 1)
        assert np.abs(d.reshape(-1) - wi).max() <= 1e-9 * max(1.0, np.abs(wi).max()), (i, j, fl[i])
        assert abs(vi - vj) <= 1e-9 * m.sill
