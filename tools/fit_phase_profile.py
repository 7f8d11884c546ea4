"""Per-phase cycle counts of the device TRF (library built with
VK_NVCC_EXTRA=-DVK_FIT_PROFILE).  Development tool."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2303_09523_b200 import ZPartKriging, _lib
from paper_2303_09523_b200.phantoms import CONFIGS, phantom_planes
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
ks = phantom_planes(cfg, cfg.known_z)
zk = ZPartKriging(cfg.n_known, cfg.height, cfg.width, cfg.factor, cfg.n_subparts, overlap=False)
kd = torch.from_numpy(ks).cuda()
lib = _lib.load()
buf = (C.c_ulonglong * 16)()
zk.run(kd); zk.finish()
lib.vk_debug_fit_profile(buf, 1)
zk.run(kd); zk.finish()
lib.vk_debug_fit_profile(buf, 0)
names = ["resid", "jac+grad", "svd", "lsq", "select", "total", "iterations", "nfev"]
tot = buf[5]
for i, n in enumerate(names):
    if i < 6: print(f"{n:10s} {buf[i]/1e6:10.2f} Mcycles ({100*buf[i]/tot:5.1f}%)")
    else: print(f"{n:10s} {buf[i]}")
for i, n in zip(range(8, 16), ["svd dgeqr2", "svd dorg2r", "svd dormbr x2", "svd dgemm+out", "svd dgebd2", "svd dbdsdc",
                               "  dnrm2 (warp)", "  dgeqr2 dlarf"]):
    print(f"{n:14s} {buf[i]/1e6:10.2f} Mcycles ({100*buf[i]/tot:5.1f}%)")
print(f"cycles per iteration {tot/buf[6]:.0f} (summed over {cfg.n_subparts} parts)")
