"""CPU evidence for the end-to-end fit tolerance:
the reference algorithm itself moves by more than 1e-6 of the range when only
libm's exp changes at the ulp level, because scipy's TRF stops on ftol inside
a flat valley.  The device fit is held to FIT_FUZZ = 5e-5 for that reason;
the kriging with given models is held to 1e-6."""

import math

import numpy as np

from oracle import kriging_oracle as O
from paper_2303_09523_b200.phantoms import known_slices, small_config


def test_reference_is_not_reproducible_below_1e6_under_exp_changes(monkeypatch):
    cfg = small_config("head", 40, 200, 9, 4, n_subparts=2, seed=7)
    ks = known_slices(cfg)
    ref, _, _ = O.reconstruct_zparts(ks, cfg.factor, cfg.n_subparts)
    vexp = np.vectorize(math.exp)

    def glibc_semivariance(self, h):
        lag = np.asarray(h, dtype=np.float64)
        partial = self.sill - self.nugget
        shape = 1.0 - vexp(-3.0 * lag / self.range_len)
        return np.where(lag == 0.0, 0.0, self.nugget + partial * shape)

    monkeypatch.setattr(O.Model, "semivariance", glibc_semivariance)
    alt, _, _ = O.reconstruct_zparts(ks, cfg.factor, cfg.n_subparts)
    fuzz = np.abs(ref.astype(np.float64) - alt).max() / float(ks.max() - ks.min())
    assert 1e-6 < fuzz < 5e-5, fuzz
