"""One C4 execute (serial schedule) for profiling the stage kernels under ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2303_09523_b200 import ZPartKriging
from paper_2303_09523_b200.phantoms import CONFIGS, phantom_planes
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = CONFIGS[name]
ks = phantom_planes(cfg, cfg.known_z)
zk = ZPartKriging(cfg.n_known, cfg.height, cfg.width, cfg.factor, cfg.n_subparts, overlap=False, redraw_pairs=True)
kd = torch.from_numpy(ks).cuda()
for _ in range(2):
    out, _ = zk.run(kd)
    models, _ = zk.finish()
torch.cuda.synchronize()
print("ok", models[0])
