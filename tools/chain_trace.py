"""Per-part timeline of the chained schedule (debug): runs the C4 path a few
times with VK_CHAIN_TRACE=1, which makes vk_plan_execute print, per part, the
completion time of its fit, solve and predict relative to the fork.

    CUDA_DEVICE_MAX_CONNECTIONS=32 VK_CHAIN_TRACE=1 python tools/chain_trace.py
"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2303_09523_b200 import ZPartKriging
from paper_2303_09523_b200.phantoms import CONFIGS, known_slices
cfg = CONFIGS["C4"]
ks = torch.from_numpy(known_slices(cfg)).cuda()
zk = ZPartKriging(cfg.n_known, cfg.height, cfg.width, cfg.factor, cfg.n_subparts, redraw_pairs=True, part_len=cfg.n_known // cfg.n_subparts)
for i in range(4):
    zk.run(ks); zk.finish()
    print("---", flush=True)
