"""CPU: the oracle's solve (oracle/kriging_oracle.py solve, restating
kriging.py:200-245) against the live reference's recovery-path goldens
(tests/golden/make_golden_ridge.py): same branch (first solve accepted /
ridge retry / SingularSystem), same weights and variance."""

import json
import os

import numpy as np
import pytest

from oracle import kriging_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
META = json.load(open(os.path.join(HERE, "golden", "reference_ridge.json")))
GOLD = np.load(os.path.join(HERE, "golden", "reference_ridge.npz"))


def test_goldens_cover_every_branch():
    outcomes = {c["outcome"] for c in META["cases"]}
    assert outcomes == {"ok", "ridge", "singular"}


@pytest.mark.parametrize("case", META["cases"], ids=lambda c: c["name"])
def test_oracle_recovery_path(case):
    import warnings
    warnings.filterwarnings("ignore")
    rel = GOLD[f"{case['name']}_rel"]
    model = O.Model(case["kind"], *case["model"])
    args = O.assemble(rel, model, case["drift"])
    if case["outcome"] == "singular":
        with pytest.raises(O.SingularSystem):
            O.solve(*args)
        return
    w, _, var, ridged = O.solve(*args)
    assert ridged == (case["outcome"] == "ridge")
    ref = GOLD[f"{case['name']}_w"]
    assert np.array_equal(w, ref)
    assert var == case["variance"]
