"""Debug: per-phase cycle counts of the device TRF fit (build with
VK_NVCC_EXTRA=-DVK_FIT_PROFILE).  Prints average cycles per part."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_09523_b200 import ZPartKriging, _lib  # noqa: E402
from paper_2303_09523_b200.phantoms import CONFIGS, known_slices  # noqa: E402

cfg = CONFIGS["C4"]
ks = torch.from_numpy(known_slices(cfg)).cuda()
zk = ZPartKriging(cfg.n_known, cfg.height, cfg.width, cfg.factor, cfg.n_subparts)
lib = _lib.load()
fn = lib.vk_debug_fit_profile
fn.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(12, np.uint64)
zk.run(ks)
zk.finish()
fn(buf.ctypes.data, 1)
zk.run(ks)
zk.finish()
fn(buf.ctypes.data, 1)
names = ["jac+grad", "svd_uf", "trust_region", "select_step", "resid", "total", "nfev", "iters",
         "svd: qr", "svd: jacobi", "jacobi sweeps"]
S = cfg.n_subparts
for n, v in zip(names, buf):
    print(f"{n:14s} {int(v) / S:12.0f} per part")
