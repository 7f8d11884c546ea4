"""Golden variogram fits of every Z sub-part of the five BASELINE configs,
produced by the LIVE reference (volkrig, read-only at /root/reference/pkg/src).
Run in the build container only:

    python tests/golden/make_golden_fits.py            # C1..C5
    python tests/golden/make_golden_fits.py C1 C2      # a subset (merged)

For each part of each config the fixture keeps
  * the reference's fitted (nugget, sill, range_len) -- kriging.py:264-328 via
    ``volkrig.kriging.fit_variogram`` on the part's samples (x, y, z coords of
    the known voxels in np.nonzero order), kind exponential, seed 0;
  * scipy's TRF bookkeeping for that fit (status, nfev, njev) and its cost;
  * the empirical bins the fit consumed (counts, sums of 0.5 dv^2, hmax, svar),
    so the CPU suite can check the TRF restatement without phantoms;
  * sha256 of the config's known slices, so a GPU box can assert that it
    regenerated bit-identical inputs before comparing fits.

This pins parity for A10 (fit_variogram) at SURVEY Appendix A.5's gate on the
full-size configs.  The arithmetic these numbers carry is the reference's as
run here: numpy 2.3.5 np.exp dispatched to SVML exp8_ha (AVX512_SKX) and
OpenBLAS 0.3.30 SKYLAKEX kernels -- see DESIGN.md "Fit parity".
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np
import scipy
import scipy.optimize

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)

from volkrig import kriging as K         # noqa: E402

from oracle import kriging_oracle as O   # noqa: E402  (bins only)
from paper_2303_09523_b200.phantoms import CONFIGS, known_slices  # noqa: E402

OUT = os.path.join(HERE, "reference_fits.json")


def _env():
    import numpy.__config__ as npc
    from numpy._core._multiarray_umath import __cpu_features__ as feat
    blas = npc.CONFIG.get("Build Dependencies", {}).get("blas", {})
    return {"numpy": np.__version__, "scipy": scipy.__version__,
            "blas": f"{blas.get('name')} {blas.get('version')}",
            "avx512_skx": bool(feat.get("AVX512_SKX"))}


def _capture():
    """Wrap scipy.optimize.least_squares so the fit's OptimizeResult is kept."""
    box = {}
    orig = scipy.optimize.least_squares

    def wrapped(*a, **k):
        r = orig(*a, **k)
        box["res"] = r
        return r
    scipy.optimize.least_squares = wrapped
    return box, orig


def run(names):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {"env": _env(), "configs": {}}
    data["env"] = _env()
    box, orig = _capture()
    try:
        for name in names:
            cfg = CONFIGS[name]
            t0 = time.time()
            ks = known_slices(cfg)
            sha = hashlib.sha256(np.ascontiguousarray(ks).tobytes()).hexdigest()
            parts = []
            for s, (b, e) in enumerate(O.subpart_ranges(cfg.n_known, cfg.n_subparts)):
                d, m = O.subpart_grid(ks, b, e, cfg.factor)
                c, v = O.subpart_samples(d, m)
                mdl = K.fit_variogram((c, v), "exponential", seed=0)
                res = box.pop("res")
                bins = O.empirical_bins(c, v)
                parts.append({
                    "part": s, "b": b, "e": e, "m": int(len(v)),
                    "nugget": mdl.nugget, "sill": mdl.sill, "range_len": mdl.range_len,
                    "x": [float(t) for t in res.x], "status": int(res.status),
                    "nfev": int(res.nfev), "njev": int(res.njev or 0), "cost": float(res.cost),
                    "counts": [int(t) for t in bins.counts],
                    "sums": [float(t).hex() for t in bins.sums],
                    "hmax": float(bins.hmax).hex(), "svar": float(bins.svar).hex(),
                })
                del d, m, c, v
            data["configs"][name] = {"sha256": sha, "shape": list(ks.shape),
                                     "factor": cfg.factor, "n_subparts": cfg.n_subparts,
                                     "parts": parts}
            print(f"{name}: {len(parts)} parts in {time.time() - t0:.1f} s", flush=True)
            del ks
            json.dump(data, open(OUT, "w"), indent=1)
    finally:
        scipy.optimize.least_squares = orig


if __name__ == "__main__":
    run(sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"])
