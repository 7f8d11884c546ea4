"""GPU: the device solves (vk_solve_systems, the batched CTA LU of
vk_generic.cu, and the stencil warp LU of vk_solve.cu through the Z-part
path) on the live reference's recovery-path goldens (kriging.py:200-245,
tests/golden/make_golden_ridge.py): systems whose first solve the reference
rejects and retries with the ridge, systems it accepts, and the one it
rejects twice (SingularSystem).  Weights and variance are held to the
solve's rounding: 1e-9 relative, scaled by the final matrix's condition
number where that is larger."""

import json
import os
import warnings

import numpy as np
import pytest

from oracle import kriging_oracle as O

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
META = json.load(open(os.path.join(HERE, "golden", "reference_ridge.json")))
GOLD = np.load(os.path.join(HERE, "golden", "reference_ridge.npz"))


def _cond(case, rel, model):
    warnings.filterwarnings("ignore")
    A, b, n, Q, q0 = O.assemble(rel, model, case["drift"])
    if case["outcome"] == "ridge":
        A = A.copy()
        A[:n, :n] += max(1e-10 * np.trace(A[:n, :n]) / n, 1e-12) * np.eye(n)
    return float(np.linalg.cond(A))


@pytest.mark.parametrize("case", META["cases"], ids=lambda c: c["name"])
def test_device_recovery_path(cuda, case):
    from paper_2303_09523_b200 import SingularSystem, VariogramModel, solve_systems
    rel = GOLD[f"{case['name']}_rel"]
    model = VariogramModel(case["kind"], *case["model"])
    if case["outcome"] == "singular":
        with pytest.raises(SingularSystem):
            solve_systems([rel], model, case["drift"])
        return
    ws, vs = solve_systems([rel], model, case["drift"])
    ref = GOLD[f"{case['name']}_w"]
    cond = _cond(case, rel, O.Model(case["kind"], *case["model"]))
    tol = max(1e-9, 1e2 * np.finfo(float).eps * cond)
    err = float(np.abs(ws[0] - ref).max() / max(1.0, np.abs(ref).max()))
    # the variance is a difference of O(sill) terms: its error is relative to the sill
    verr = abs(vs[0] - case["variance"]) / max(abs(case["variance"]), case["model"][1], 1e-300)
    print(f"\n{case['name']} {case['outcome']} cond {cond:.1e} w err {err:.2e} var err {verr:.2e}")
    assert err <= tol
    assert verr <= max(tol, 1e-9)
