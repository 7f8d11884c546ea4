"""Per-chain completion times of one C4 execute on the default (chained)
schedule (VK_CHAIN_TRACE), after warm-up.  Development tool."""
import os, sys
os.environ["CUDA_DEVICE_MAX_CONNECTIONS"] = "32"
os.environ["VK_CHAIN_TRACE"] = "1"      # read once, at the first execute (the last block printed counts)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_09523_b200 import ZPartKriging
from paper_2303_09523_b200.phantoms import CONFIGS, phantom_planes
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
ks = phantom_planes(cfg, cfg.known_z)
zk = ZPartKriging(cfg.n_known, cfg.height, cfg.width, cfg.factor, cfg.n_subparts, redraw_pairs=True)
kd = torch.from_numpy(ks).cuda()
for _ in range(3):
    zk.run(kd); zk.finish()
zk.run(kd); zk.finish()
