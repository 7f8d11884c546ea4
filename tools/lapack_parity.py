"""Component check of csrc/gesdd.h (via the test shim) against the LAPACK/BLAS
routines of the OpenBLAS that numpy ships (called directly through ctypes).
Development tool: prints mismatch counts per routine on random inputs."""
import ctypes as C, glob, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import native_build
S = native_build.build_shim()
OB = C.CDLL(glob.glob(os.path.join(os.path.dirname(np.__file__) + ".libs", "libscipy_openblas64_*.so"))[0])
I = C.c_int64; D = C.c_double
def ip(v): return C.byref(I(v))
def dp(a): return a.ctypes.data_as(C.POINTER(C.c_double))
def ch(s): return C.c_char_p(s.encode())
ONE = C.c_size_t(1)
OB.scipy_dnrm2_64_.restype = D
S.vkl_dnrm2.restype = D
S.vkl_dlarf.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, D, C.c_void_p, C.c_int]
S.vkl_dlartg.argtypes = [D, D, C.c_void_p, C.c_void_p, C.c_void_p]
S.vkl_dlas2.argtypes = [D, D, D, C.c_void_p, C.c_void_p]
S.vkl_dlasv2.argtypes = [D, D, D, C.c_void_p]
S.vkl_drot.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, D, D]
S.vkl_dger.argtypes = [C.c_int, C.c_int, D, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int]
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
def rv(n, spread=6):
    return rng.standard_normal(n) * np.exp(rng.uniform(-spread, spread, n))
def report(name, bad, tot): print(f"{name:10s} mismatches {bad}/{tot}")
def eq(a, b): return np.array_equal(np.asarray(a), np.asarray(b))

bad = 0
for t in range(20000):
    n = int(rng.integers(1, 36)); x = rv(n, 3)
    bad += OB.scipy_dnrm2_64_(ip(n), dp(x), ip(1)) != S.vkl_dnrm2(n, dp(x), 1)
report("dnrm2", bad, 20000)

bad = 0
for t in range(5000):
    n = int(rng.integers(2, 20)); x = rv(n - 1); a = np.array([rv(1)[0]])
    x2, a2 = x.copy(), a.copy(); tau1 = np.zeros(1); tau2 = np.zeros(1)
    OB.scipy_dlarfg_64_(ip(n), dp(a), dp(x), ip(1), dp(tau1))
    S.vkl_dlarfg(n, dp(a2), dp(x2), 1, dp(tau2))
    bad += not (eq(x, x2) and eq(a, a2) and eq(tau1, tau2))
report("dlarfg", bad, 5000)

bad = 0
for t in range(5000):
    f, g = rv(2, 10); c1, s1, r1 = D(), D(), D(); c2, s2, r2 = D(), D(), D()
    OB.scipy_dlartg_64_(C.byref(D(f)), C.byref(D(g)), C.byref(c1), C.byref(s1), C.byref(r1))
    S.vkl_dlartg(f, g, C.byref(c2), C.byref(s2), C.byref(r2))
    bad += (c1.value, s1.value, r1.value) != (c2.value, s2.value, r2.value)
report("dlartg", bad, 5000)

bad = 0
for t in range(5000):
    f, g, h = rv(3, 8); a1, b1 = D(), D(); a2, b2 = D(), D()
    OB.scipy_dlas2_64_(C.byref(D(f)), C.byref(D(g)), C.byref(D(h)), C.byref(a1), C.byref(b1))
    S.vkl_dlas2(f, g, h, C.byref(a2), C.byref(b2))
    bad += (a1.value, b1.value) != (a2.value, b2.value)
report("dlas2", bad, 5000)

bad = 0
for t in range(5000):
    f, g, h = rv(3, 8); o1 = [D() for _ in range(6)]; o2 = np.zeros(6)
    OB.scipy_dlasv2_64_(C.byref(D(f)), C.byref(D(g)), C.byref(D(h)), *[C.byref(o) for o in o1])
    S.vkl_dlasv2(f, g, h, o2.ctypes.data)
    bad += [o.value for o in o1] != list(o2)
report("dlasv2", bad, 5000)

bad = 0
for t in range(3000):
    n = int(rng.integers(1, 6)); x = rv(n); y = rv(n); c, s = rng.uniform(-1, 1, 2)
    x2, y2 = x.copy(), y.copy()
    OB.scipy_drot_64_(ip(n), dp(x), ip(1), dp(y), ip(1), C.byref(D(c)), C.byref(D(s)))
    S.vkl_drot(n, x2.ctypes.data, 1, y2.ctypes.data, 1, c, s)
    bad += not (eq(x, x2) and eq(y, y2))
report("drot", bad, 3000)

bad = 0
for t in range(3000):
    m = int(rng.integers(1, 20)); n = int(rng.integers(1, 4)); A = np.asfortranarray(rv(m * n).reshape(m, n))
    x = rv(m); y = rv(n); al = rv(1)[0]; A2 = A.copy(order="F")
    OB.scipy_dger_64_(ip(m), ip(n), C.byref(D(al)), dp(x), ip(1), dp(y), ip(1), dp(A), ip(m))
    S.vkl_dger(m, n, al, x.ctypes.data, y.ctypes.data, 1, A2.ctypes.data, m)
    bad += not eq(A, A2)
report("dger", bad, 3000)

bad = 0
for t in range(3000):
    m = int(rng.integers(1, 20)); n = int(rng.integers(1, 4)); A = np.asfortranarray(rv(m * n).reshape(m, n))
    x = rv(m); y1 = np.zeros(n); y2 = np.zeros(n)
    OB.scipy_dgemv_64_(ch("T"), ip(m), ip(n), C.byref(D(1.0)), dp(A), ip(m), dp(x), ip(1), C.byref(D(0.0)), dp(y1), ip(1), ONE)
    S.vkl_dgemv_t(m, n, dp(A), m, dp(x), dp(y2))
    bad += not eq(y1, y2)
report("dgemv_t", bad, 3000)

bad = 0
for t in range(3000):
    m = int(rng.integers(1, 4)); n = int(rng.integers(1, 4)); lda = 3; incx = int(rng.choice([1, 3]))
    A = np.asfortranarray(rv(lda * n).reshape(lda, n)); x = rv(n * incx); y1 = np.zeros(m); y2 = np.zeros(m)
    OB.scipy_dgemv_64_(ch("N"), ip(m), ip(n), C.byref(D(1.0)), dp(A), ip(lda), dp(x), ip(incx), C.byref(D(0.0)), dp(y1), ip(1), ONE)
    S.vkl_dgemv_n(m, n, dp(A), lda, dp(x), incx, dp(y2))
    bad += not eq(y1, y2)
report("dgemv_n", bad, 3000)

def lapack_qr(A):
    m, n = A.shape; a = np.asfortranarray(A.copy()); tau = np.zeros(n); w = np.zeros(64); info = I(0)
    OB.scipy_dgeqr2_64_(ip(m), ip(n), dp(a), ip(m), dp(tau), dp(w), C.byref(info))
    return a, tau
bad = 0
for t in range(3000):
    m = int(rng.integers(5, 36)); A = rv(m * 3).reshape(m, 3)
    a1, t1 = lapack_qr(A); a2 = np.asfortranarray(A.copy()); t2 = np.zeros(3)
    S.vkl_dgeqr2(m, 3, dp(a2), m, dp(t2))
    bad += not (eq(a1, a2) and eq(t1, t2))
report("dgeqr2", bad, 3000)

bad = 0
for t in range(3000):
    m = int(rng.integers(5, 36)); A = rv(m * 3).reshape(m, 3)
    a1, t1 = lapack_qr(A); a2 = a1.copy(order="F"); w = np.zeros(64); info = I(0)
    OB.scipy_dorg2r_64_(ip(m), ip(3), ip(3), dp(a1), ip(m), dp(t1), dp(w), C.byref(info))
    S.vkl_dorg2r(m, 3, 3, dp(a2), m, dp(t1))
    bad += not eq(a1, a2)
report("dorg2r", bad, 3000)

bad = 0
for t in range(3000):
    R = np.asfortranarray(np.triu(rv(9).reshape(3, 3))); R2 = R.copy(order="F")
    d1, e1, q1, p1 = np.zeros(3), np.zeros(3), np.zeros(3), np.zeros(3)
    d2, e2, q2, p2 = np.zeros(3), np.zeros(3), np.zeros(3), np.zeros(3); w = np.zeros(64); info = I(0)
    OB.scipy_dgebd2_64_(ip(3), ip(3), dp(R), ip(3), dp(d1), dp(e1), dp(q1), dp(p1), dp(w), C.byref(info))
    S.vkl_dgebd2(3, 3, dp(R2), 3, dp(d2), dp(e2), dp(q2), dp(p2))
    bad += not (eq(R, R2) and eq(d1, d2) and eq(e1[:2], e2[:2]) and eq(q1, q2) and eq(p1, p2))
report("dgebd2", bad, 3000)

bad = 0; binfo = 0
for t in range(5000):
    d = rv(3, 4); e = rv(3, 4); e[2] = 0
    if t % 5 == 1: e[0] *= 1e-9
    if t % 5 == 2: d[2] *= 1e-12
    d1, e1, d2, e2 = d.copy(), e.copy(), d.copy(), e.copy()
    U1 = np.zeros((3, 3), order="F"); VT1 = np.zeros((3, 3), order="F"); U2 = U1.copy(order="F"); VT2 = VT1.copy(order="F")
    w = np.zeros(64); iw = np.zeros(64, np.int64); info = I(0); dum = np.zeros(1); idum = np.zeros(1, np.int64)
    OB.scipy_dbdsdc_64_(ch("U"), ch("I"), ip(3), dp(d1), dp(e1), dp(U1), ip(3), dp(VT1), ip(3), dp(dum), idum.ctypes.data_as(C.POINTER(I)), dp(w), iw.ctypes.data_as(C.POINTER(I)), C.byref(info), ONE, ONE)
    r = S.vkl_dbdsdc(3, dp(d2), dp(e2), dp(U2), 3, dp(VT2), 3)
    ok = eq(d1, d2) and eq(U1, U2) and eq(VT1, VT2)
    bad += not ok
report("dbdsdc", bad, 5000)

bad = 0
for t in range(5000):
    m = int(rng.integers(5, 19)); A = rv(m * 3).reshape(m, 3)
    if t % 2: A[m - 3:] = np.diag(np.abs(rv(3)))
    U1, s1, VT1 = np.linalg.svd(A, full_matrices=False)
    U2 = np.zeros((m, 3)); s2 = np.zeros(3); VT2 = np.zeros((3, 3)); Ac = np.ascontiguousarray(A)
    S.vkl_svd_m3(dp(Ac), m, dp(U2), dp(s2), dp(VT2))
    bad += not (eq(U1, U2) and eq(s1, s2) and eq(VT1, VT2))
report("svd", bad, 5000)
