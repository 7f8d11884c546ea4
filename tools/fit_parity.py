"""Host TRF restatement (trf.h via the test shim) against the live reference's
fits of every part of C1..C5 (tests/golden/reference_fits.json), in SURVEY
Appendix A.5 gate units.  Development tool (CPU only)."""
import json, os, sys
import ctypes as C
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests")); sys.path.insert(0, ROOT)
import native_build
D = C.POINTER(C.c_double); I32 = C.POINTER(C.c_int32)
shim = native_build.build_shim()
G = json.load(open(os.path.join(ROOT, "tests/golden/reference_fits.json")))
worst = 0
for name, cfg in G["configs"].items():
    for p in cfg["parts"]:
        counts = np.array(p["counts"]); sums = np.array([float.fromhex(s) for s in p["sums"]])
        hmax = float.fromhex(p["hmax"]); svar = float.fromhex(p["svar"])
        edges = np.linspace(0.0, hmax, 16); nz = counts > 0
        h = np.ascontiguousarray((0.5 * (edges[:-1] + edges[1:]))[nz]); g = np.ascontiguousarray(sums[nz] / counts[nz])
        w = np.ascontiguousarray(np.sqrt(counts[nz].astype(float)))
        x0 = np.array([0.0, svar, hmax / 3]); lb = np.array([0.0, 0.0, 1e-6])
        ub = np.array([2 * svar + 1e-12, 4 * svar + 1e-12, 10 * hmax])
        x = np.zeros(3); info = np.zeros(3, np.int32)
        shim.vkh_trf(0, len(h), h.ctypes.data_as(D), g.ctypes.data_as(D), w.ctypes.data_as(D),
                     x0.ctypes.data_as(D), lb.ctypes.data_as(D), ub.ctypes.data_as(D),
                     x.ctypes.data_as(D), info.ctypes.data_as(I32))
        nug = max(x[0], 0.0); sill = nug + max(x[1], 0.0); rng = max(x[2], 1e-6)
        dn = abs(nug - p["nugget"]) / p["sill"] / 1e-7
        ds = abs(sill - p["sill"]) / p["sill"] / 1e-6
        dr = abs(rng - p["range_len"]) / p["range_len"] / 1e-4
        gate = max(dn, ds, dr); worst = max(worst, gate)
        exact = (x.tolist() == p["x"])
        flag = "EXACT" if exact else ("ok" if gate <= 1 else "MISS")
        if "-v" in sys.argv or flag == "MISS":
            print(f"{name} p{p['part']:2d} nfev {info[1]:3d}/{p['nfev']:3d} st {info[0]}/{p['status']} "
                  f"gate nug {dn:9.3g} sill {ds:9.3g} rng {dr:9.3g} {flag}")
print("worst gate ratio", worst)
