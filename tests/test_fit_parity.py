"""CPU: the restated arithmetic of the reference's variogram fit (what the
device runs, compiled for the host through tests/native/host_shim.cpp)
against the numpy / scipy / OpenBLAS the reference runs on, and the whole
host TRF against the live reference's fits of every part of C1-C5.

kriging.py:264-328 reaches, through numpy 2.3.5 and scipy 1.18.1:
  np.exp                -> SVML exp8_ha (AVX512_SKX hosts)      npref.h exp_
  np.dot / J.dot / J.T  -> OpenBLAS 0.3.30 ddot / dgemv SKYLAKEX npref.h dot/row3/colT/rowN
  numpy.linalg.svd      -> LAPACK dgesdd (dnrm2 in x87)         gesdd.h
  values.var()          -> numpy pairwise summation             npsum.h
Each piece is compared bit for bit on random inputs; the full host TRF must
reproduce scipy's fit bit for bit on every part except the CUBE_PARTS (x**3
through SVML pow8_ha, restated as the correctly rounded cube), which stay
far inside SURVEY Appendix A.5's gate.
"""

import ctypes as C
import glob
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
D = C.POINTER(C.c_double)
I32 = C.POINTER(C.c_int32)
CUBE_PARTS = {("C3", 2), ("C3", 14), ("C4", 25)}


@pytest.fixture(scope="module")
def shim():
    import native_build
    s = native_build.build_shim()
    s.vkl_dnrm2.restype = C.c_double
    s.vkh_npsum_tree.restype = C.c_double
    s.vkl_dlartg.argtypes = [C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
    s.vkl_dlasv2.argtypes = [C.c_double, C.c_double, C.c_double, C.c_void_p]
    return s


@pytest.fixture(scope="module")
def openblas():
    libs = glob.glob(os.path.join(os.path.dirname(np.__file__) + ".libs", "libscipy_openblas64_*.so"))
    if not libs:
        pytest.skip("numpy's bundled OpenBLAS not found")
    L = C.CDLL(libs[0])
    L.scipy_dnrm2_64_.restype = C.c_double
    cfg = ""
    if hasattr(L, "scipy_openblas_get_config64_"):
        L.scipy_openblas_get_config64_.restype = C.c_char_p
        cfg = L.scipy_openblas_get_config64_().decode()
    if "SkylakeX" not in cfg:
        pytest.skip(f"OpenBLAS core is not SkylakeX ({cfg}): the restated kernel orders are SKYLAKEX's")
    return L


def _rv(rng, n, spread=6):
    return rng.standard_normal(n) * np.exp(rng.uniform(-spread, spread, n))


def test_exp_is_numpys(shim):
    from numpy._core._multiarray_umath import __cpu_features__ as feat
    if not feat.get("AVX512_SKX"):
        pytest.skip("np.exp dispatches to SVML exp8_ha only on AVX512_SKX hosts")
    rng = np.random.default_rng(0)
    x = np.concatenate([-rng.uniform(0, 50, 400_000), -rng.exponential(2, 200_000),
                        rng.uniform(-700, 700, 50_000), -rng.uniform(0, 1e-8, 10_000), [0.0, -0.0]])
    y = np.empty_like(x)
    shim.vkh_np_exp(x.ctypes.data_as(D), y.ctypes.data_as(D), C.c_long(len(x)))
    assert np.array_equal(y, np.exp(x))


def test_blas_orders_are_openblas(shim, openblas):
    """np.dot (n < 16), J.dot(s) (C order), J.T.dot(f) (F order), U.T.dot(f)
    (dgemv_n, 3 rows) as the host TRF forms them (through its LAPACK-side
    dgemv_t / dgemv_n restatements, same kernels)."""
    rng = np.random.default_rng(1)
    for m in range(1, 19):
        for _ in range(60):
            J = np.asfortranarray(_rv(rng, 3 * m).reshape(m, 3))
            f = _rv(rng, m)
            y = np.zeros(3)
            shim.vkl_dgemv_t(m, 3, J.ctypes.data_as(D), m, f.ctypes.data_as(D), y.ctypes.data_as(D))
            assert np.array_equal(y, J.T.dot(f)), m
            U = np.ascontiguousarray(_rv(rng, 3 * m).reshape(m, 3))
            y2 = np.zeros(3)
            # U.T is an F-ordered (3, m) matrix: dgemv_n with lda = 3, incx = 1
            shim.vkl_dgemv_n(3, m, U.ctypes.data_as(D), 3, f.ctypes.data_as(D), 1, y2.ctypes.data_as(D))
            assert np.array_equal(y2, U.T.dot(f)), m


def test_lapack_pieces_are_openblas(shim, openblas):
    L = openblas
    I = C.c_int64
    rng = np.random.default_rng(2)

    def ip(v):
        return C.byref(I(v))

    for _ in range(2000):
        n = int(rng.integers(1, 36))
        x = _rv(rng, n, 3)
        assert L.scipy_dnrm2_64_(ip(n), x.ctypes.data_as(D), ip(1)) == shim.vkl_dnrm2(n, x.ctypes.data_as(D), 1)
    for _ in range(1000):
        f, g = _rv(rng, 2, 10)
        c1, s1, r1, c2, s2, r2 = (C.c_double() for _ in range(6))
        L.scipy_dlartg_64_(C.byref(C.c_double(f)), C.byref(C.c_double(g)), C.byref(c1), C.byref(s1), C.byref(r1))
        shim.vkl_dlartg(f, g, C.byref(c2), C.byref(s2), C.byref(r2))
        assert (c1.value, s1.value, r1.value) == (c2.value, s2.value, r2.value)
    for _ in range(1000):
        f, g, h = _rv(rng, 3, 8)
        o1 = [C.c_double() for _ in range(6)]
        o2 = np.zeros(6)
        L.scipy_dlasv2_64_(C.byref(C.c_double(f)), C.byref(C.c_double(g)), C.byref(C.c_double(h)),
                           *[C.byref(o) for o in o1])
        shim.vkl_dlasv2(f, g, h, o2.ctypes.data)
        assert [o.value for o in o1] == list(o2)
    for t in range(3000):
        # random bidiagonals plus the structures that take dbdsqr's other
        # branches: zero / tiny off-diagonals (splits, 2 x 2 blocks), zero
        # diagonal entries, graded magnitudes (zero shift, both directions)
        d = _rv(rng, 3, 4)
        e = _rv(rng, 3, 4)
        e[2] = 0
        k = t % 6
        if k == 1:
            e[rng.integers(0, 2)] *= 1e-18
        elif k == 2:
            d[rng.integers(0, 3)] = 0.0
        elif k == 3:
            d *= np.array([1e-9, 1.0, 1e9])[rng.permutation(3)]
        elif k == 4:
            e[rng.integers(0, 2)] = 0.0
        elif k == 5:
            d = np.round(d * 4) / 4
            e = np.round(e * 4) / 4
            e[2] = 0
        d1, e1, d2, e2 = d.copy(), e.copy(), d.copy(), e.copy()
        U1 = np.zeros((3, 3), order="F"); V1 = np.zeros((3, 3), order="F")
        U2 = np.zeros((3, 3), order="F"); V2 = np.zeros((3, 3), order="F")
        w = np.zeros(64); iw = np.zeros(64, np.int64); info = I(0)
        dum = np.zeros(1); idum = np.zeros(1, np.int64); one = C.c_size_t(1)
        L.scipy_dbdsdc_64_(C.c_char_p(b"U"), C.c_char_p(b"I"), ip(3), d1.ctypes.data_as(D), e1.ctypes.data_as(D),
                           U1.ctypes.data_as(D), ip(3), V1.ctypes.data_as(D), ip(3), dum.ctypes.data_as(D),
                           idum.ctypes.data_as(C.POINTER(I)), w.ctypes.data_as(D),
                           iw.ctypes.data_as(C.POINTER(I)), C.byref(info), one, one)
        shim.vkl_dbdsdc(3, d2.ctypes.data_as(D), e2.ctypes.data_as(D), U2.ctypes.data_as(D), 3,
                        V2.ctypes.data_as(D), 3)
        assert np.array_equal(d1, d2) and np.array_equal(U1, U2) and np.array_equal(V1, V2)


def test_svd_is_numpys(shim, openblas):
    rng = np.random.default_rng(3)
    for t in range(1500):
        m = int(rng.integers(5, 36))
        A = _rv(rng, 3 * m).reshape(m, 3)
        if t % 2:
            A[m - 3:] = np.diag(np.abs(_rv(rng, 3)))           # augmented-Jacobian shape
        U1, s1, V1 = np.linalg.svd(A, full_matrices=False)
        U2 = np.zeros((m, 3)); s2 = np.zeros(3); V2 = np.zeros((3, 3))
        A = np.ascontiguousarray(A)
        assert shim.vkl_svd_m3(A.ctypes.data_as(D), m, U2.ctypes.data_as(D), s2.ctypes.data_as(D),
                               V2.ctypes.data_as(D)) == 0
        assert np.array_equal(U1, U2) and np.array_equal(s1, s2) and np.array_equal(V1, V2), t


def test_pairwise_sum_tree_is_numpys(shim):
    rng = np.random.default_rng(4)
    for n in list(rng.integers(9, 4000, 40)) + [8191, 81920, 327680, 2359296]:
        a = rng.standard_normal(int(n)) * 1e3 + rng.uniform(0, 50)
        nl = C.c_int32(0)
        assert shim.vkh_npsum_tree(a.ctypes.data_as(D), C.c_int64(len(a)), C.byref(nl)) == a.sum(), n
        t = (a - a.mean()) ** 2
        assert shim.vkh_npsum_tree(t.ctypes.data_as(D), C.c_int64(len(t)), C.byref(nl)) / len(a) == a.var(), n


def test_pairwise_sum_warp_decomposition_is_numpys(shim):
    """npsum.h build_npsum_warp (the device's warp subtrees + top tree) gives
    np.sum / np.var bit for bit, including sizes whose root is a leaf and the
    C1-C5 part sizes."""
    shim.vkh_npsum_warp.restype = C.c_double
    rng = np.random.default_rng(5)
    sizes = list(rng.integers(9, 5000, 60)) + [9, 100, 128, 129, 4095, 4096, 4097, 8191, 81920,
                                                 9 * 128 * 128, 5 * 256 * 256, 5 * 512 * 512,
                                                 9 * 512 * 512, 327680, 2359296]
    for n in sizes:
        a = rng.standard_normal(int(n)) * 1e3 + rng.uniform(0, 50)
        nw = C.c_int32(0)
        assert shim.vkh_npsum_warp(a.ctypes.data_as(D), C.c_int64(len(a)), C.byref(nw)) == a.sum(), n
        t = (a - a.mean()) ** 2
        assert shim.vkh_npsum_warp(t.ctypes.data_as(D), C.c_int64(len(t)), C.byref(nw)) / len(a) == a.var(), n
        assert 1 <= nw.value <= max(1, n // 128 + 1)


def _host_fit(shim, p):
    counts = np.array(p["counts"])
    sums = np.array([float.fromhex(s) for s in p["sums"]])
    hmax = float.fromhex(p["hmax"])
    svar = float.fromhex(p["svar"])
    edges = np.linspace(0.0, hmax, len(counts) + 1)
    nz = counts > 0
    h = np.ascontiguousarray((0.5 * (edges[:-1] + edges[1:]))[nz])
    g = np.ascontiguousarray(sums[nz] / counts[nz])
    w = np.ascontiguousarray(np.sqrt(counts[nz].astype(np.float64)))
    x0 = np.array([0.0, svar, hmax / 3.0])
    lb = np.array([0.0, 0.0, 1e-6])
    ub = np.array([2.0 * svar + 1e-12, 4.0 * svar + 1e-12, 10.0 * hmax])
    x = np.zeros(3)
    info = np.zeros(3, np.int32)
    shim.vkh_trf(0, len(h), h.ctypes.data_as(D), g.ctypes.data_as(D), w.ctypes.data_as(D),
                 x0.ctypes.data_as(D), lb.ctypes.data_as(D), ub.ctypes.data_as(D), x.ctypes.data_as(D),
                 info.ctypes.data_as(I32))
    return x, info


def test_host_trf_reproduces_reference_fits(shim):
    """Every part of C1-C5: the restated TRF on the reference's own bins."""
    G = json.load(open(os.path.join(HERE, "golden", "reference_fits.json")))
    total, exact, worst = 0, 0, 0.0
    for name, cfg in G["configs"].items():
        for p in cfg["parts"]:
            x, info = _host_fit(shim, p)
            nug = max(x[0], 0.0)
            sill = nug + max(x[1], 0.0)
            rng = max(x[2], 1e-6)
            gate = max(abs(nug - p["nugget"]) / p["sill"] / 1e-7, abs(sill - p["sill"]) / p["sill"] / 1e-6,
                       abs(rng - p["range_len"]) / p["range_len"] / 1e-4)
            worst = max(worst, gate)
            same = list(x) == p["x"]
            total += 1
            exact += same
            assert same or (name, p["part"]) in CUBE_PARTS, (name, p["part"], gate)
            assert info[1] == p["nfev"] and info[0] == p["status"], (name, p["part"])
    print(f"\nhost TRF: {exact}/{total} parts bit-identical, worst gate ratio {worst:.3g}")
    assert worst <= 0.05


def test_dnrm2_fast_decision_is_x87(shim, openblas):
    """dnrm2's double-double fast path (gesdd.h dnrm2_decide) against the
    shipped x87 kernel on many vectors: random magnitudes, integer vectors
    (exact sums, often near-exact square roots), repeated values and zeros."""
    L = openblas
    I = C.c_int64
    rng = np.random.default_rng(11)
    n_vec = 60000
    for t in range(n_vec):
        n = int(rng.integers(2, 19))
        kind = t % 4
        if kind == 0:
            x = _rv(rng, n, 8)
        elif kind == 1:
            x = rng.integers(-4096, 4096, n).astype(np.float64)
        elif kind == 2:
            x = np.full(n, _rv(rng, 1, 4)[0])
        else:
            x = _rv(rng, n, 2)
            x[rng.random(n) < 0.4] = 0.0
        got = shim.vkl_dnrm2(n, x.ctypes.data_as(D), 1)
        ref = L.scipy_dnrm2_64_(C.byref(I(n)), x.ctypes.data_as(D), C.byref(I(1)))
        assert got == ref, (t, n, x.tolist(), got, ref)
