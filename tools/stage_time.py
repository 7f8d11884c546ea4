"""Per-stage times (serial schedule) and the chained step time of one config
(development tool; bench.py is the measurement of record).

    python tools/stage_time.py [C4] [steps]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch
from paper_2303_09523_b200 import ZPartKriging
from paper_2303_09523_b200.phantoms import CONFIGS, phantom_planes

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = CONFIGS[name]
ks = torch.from_numpy(phantom_planes(cfg, cfg.known_z)).cuda()
res = {"config": name, "lib": os.environ.get("VK_VARIANT", "")}
zs = ZPartKriging(cfg.n_known, cfg.height, cfg.width, cfg.factor, cfg.n_subparts,
                  part_len=cfg.n_known // cfg.n_subparts, overlap=False, redraw_pairs=True)
out, var = zs.allocate(False)
for _ in range(3):
    zs.run(ks, out, var)
zs.finish()
zs.plan.set_timing(steps)
for _ in range(steps):
    zs.run(ks, out, var)
zs.finish()
acc = {}
for b in range(steps):
    for k, v in zs.plan.stage_ms(b).items():
        acc[k] = acc.get(k, 0.0) + v / steps
res["stage_ms"] = {k: round(v, 4) for k, v in acc.items()}
zk = ZPartKriging(cfg.n_known, cfg.height, cfg.width, cfg.factor, cfg.n_subparts,
                  part_len=cfg.n_known // cfg.n_subparts, overlap=True, redraw_pairs=True)
out, var = zk.allocate(False)
for _ in range(3):
    zk.run(ks, out, var)
zk.finish()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(steps):
    zk.run(ks, out, var)
e1.record()
torch.cuda.synchronize()
zk.finish()
res["step_ms"] = round(e0.elapsed_time(e1) / steps, 4)
print(json.dumps(res))
