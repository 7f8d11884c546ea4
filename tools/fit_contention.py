"""Fit stage time alone vs under a concurrent HBM stream on another CUDA
stream (development tool: is the chained schedule's slower fit a memory-system
effect?).   python tools/fit_contention.py [C4]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_09523_b200 import ZPartKriging
from paper_2303_09523_b200.phantoms import CONFIGS, phantom_planes

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
ks = torch.from_numpy(phantom_planes(cfg, cfg.known_z)).cuda()
zs = ZPartKriging(cfg.n_known, cfg.height, cfg.width, cfg.factor, cfg.n_subparts,
                  part_len=cfg.n_known // cfg.n_subparts, overlap=False, redraw_pairs=True)
out, var = zs.allocate(False)
src = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
dst = torch.empty_like(src)
side = torch.cuda.Stream(priority=0)
res = {}
for mode in ("alone", "hbm_copy", "alone2"):
    for _ in range(2):
        zs.run(ks, out, var)
    zs.finish()
    torch.cuda.synchronize()
    zs.plan.set_timing(5)
    for _ in range(5):
        if mode == "hbm_copy":
            with torch.cuda.stream(side):
                for _ in range(12):
                    dst.copy_(src)           # ~2 GB of HBM traffic per copy
        zs.run(ks, out, var)
    zs.finish()
    torch.cuda.synchronize()
    acc = {}
    for b in range(5):
        for k, v in zs.plan.stage_ms(b).items():
            acc[k] = acc.get(k, 0.0) + v / 5
    res[mode] = {k: round(v, 4) for k, v in acc.items()}
print(json.dumps(res))
