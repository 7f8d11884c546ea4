"""Golden vectors for solve_ked's numerical recovery path (kriging.py:200-245)
from the LIVE reference (volkrig, read-only at /root/reference/pkg/src).
Run in the build container only:

    python tests/golden/make_golden_ridge.py

Cases (integer target-relative offsets, as vk_solve_systems takes them):
  * "ridge": the first np.linalg.solve raises LinAlgError or returns a
    non-finite / constraint-violating solution, so the reference adds
    max(1e-10 * tr(C) / n, 1e-12) to the covariance block and solves again
    (duplicated neighbours, rank-deficient drift, white-noise models);
  * "ok": the first solve is accepted (including ill-conditioned gaussian
    stencils with weights in the hundreds);
  * "singular": the retry fails too and the reference raises SingularSystem
    (an infinite sill: the covariance block is inf - inf).
Each case records which branch the reference took (counted np.linalg.solve
calls), the weights and the kriging variance.
"""

from __future__ import annotations

import json
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from volkrig import errors as E          # noqa: E402
from volkrig import kriging as K         # noqa: E402


def main():
    warnings.filterwarnings("ignore")
    calls = {"n": 0}
    orig = np.linalg.solve

    def counting(a, b):
        calls["n"] += 1
        return orig(a, b)

    np.linalg.solve = counting
    cases, arrays = [], {}

    def add(name, rel, kind, nug, sill, rng_len, drift):
        rel = np.asarray(rel, np.int64).reshape(-1, 3)
        model = K.VariogramModel(kind, nug, sill, rng_len)
        calls["n"] = 0
        entry = {"name": name, "kind": kind, "model": [nug, sill, rng_len], "drift": drift}
        try:
            s = K.solve_ked(K.build_system(rel.astype(np.float64), np.zeros(len(rel)), np.zeros(3), model, drift))
            entry["outcome"] = "ridge" if calls["n"] > 1 else "ok"
            entry["variance"] = float(s.variance)
            arrays[f"{name}_w"] = s.weights
        except E.SingularSystem as ex:
            entry["outcome"] = "singular"
            entry["message"] = str(ex)
        arrays[f"{name}_rel"] = rel
        cases.append(entry)

    st = np.array([(x, y, z) for z in (-1, 2) for y in range(-1, 3) for x in range(-1, 3)])
    for drift in ("linear", "constant"):
        d = drift[:3]
        add(f"dup3_exp_{d}", np.vstack([st, st[:3]]), "exponential", 0.5, 100.0, 10.0, drift)
        add(f"dup1_white_{d}", np.vstack([st, st[:1]]), "exponential", 0.0, 0.0, 1.0, drift)
        add(f"dupall_exp_{d}", np.vstack([st, st]), "exponential", 0.0, 10.0, 5.0, drift)
        add(f"dup2_gauss_{d}", np.vstack([st, st[:2]]), "gaussian", 0.0, 100.0, 20.0, drift)
        add(f"dup_sph_{d}", np.vstack([st, st[5:7]]), "spherical", 1.0, 50.0, 30.0, drift)
        add(f"gauss_r300_{d}", st, "gaussian", 0.0, 100.0, 300.0, drift)
        add(f"infsill_{d}", st, "exponential", 0.0, float("inf"), 10.0, drift)
    rng = np.random.default_rng(20260)
    kinds = ["exponential", "gaussian", "spherical"]
    for t in range(60):
        n = int(rng.integers(2, 20))
        rel = rng.integers(-3, 4, (n, 3))
        if t % 2 == 0:
            rel = np.vstack([rel, rel[rng.integers(0, n, int(rng.integers(1, 4)))]])
        kind = kinds[t % 3]
        nug = float(rng.choice([0.0, 0.0, 1e-3, 1.0]))
        sill = nug + float(rng.choice([1.0, 100.0]))
        add(f"rand{t:02d}", rel, kind, nug, sill, float(rng.choice([0.5, 2.0, 10.0, 100.0])),
            ["linear", "constant"][t % 4 // 2])
    np.linalg.solve = orig
    np.savez_compressed(os.path.join(HERE, "reference_ridge.npz"), **arrays)
    import scipy
    json.dump({"env": {"numpy": np.__version__, "scipy": scipy.__version__}, "cases": cases},
              open(os.path.join(HERE, "reference_ridge.json"), "w"), indent=1)
    print({k: sum(c["outcome"] == k for c in cases) for k in ("ok", "ridge", "singular")})


if __name__ == "__main__":
    main()
