"""Random-shape check of the streaming kernel's unit schedule (development
tool): for each shape the serial launch (guided dynamic schedule) must write
every voxel, repeat bit for bit and equal the per-part chained launches.

    timeout 600 python tools/schedule_fuzz.py [n_cases] [seed] [big]

"big": many more (tile, gap) items than resident CTAs, so the launch has all
the schedule's levels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2303_09523_b200 import ZPartKriging

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
big = len(sys.argv) > 3 and sys.argv[3] == "big"
bad = 0
for case in range(n_cases):
    factor = int(rng.choice([2, 3, 4, 5, 8, 9]))
    parts = int(rng.integers(1, 12))
    q = int(rng.integers(1, 9))                       # known slices per part
    if big:
        parts = int(rng.integers(2, 40))
        q = int(rng.integers(2, 12))
    K = parts * q + int(rng.integers(1, 4)) if parts > 1 else int(rng.integers(2, 40))
    H = int(rng.integers(5, 200))
    W = 4 * int(rng.integers(2, 130))
    if big:
        H = int(rng.integers(100, 400))
        W = 4 * int(rng.integers(64, 160))
        while (K - 1) * factor * H * W > 120e6:       # bound the three output volumes
            H = max(64, H // 2)
            W = max(256, (W // 2) // 4 * 4)
            if H == 64 and W == 256:
                break
    accum = str(rng.choice(["fp64", "fp32"]))
    integer = bool(rng.integers(0, 2))
    var = bool(rng.integers(0, 2))
    v = rng.normal(500.0, 120.0, size=(K, H, W))
    ks = np.clip(np.rint(v), 0, 4095).astype(np.float32) if integer else (v / 4095.0).astype(np.float32)
    kd = torch.from_numpy(ks).cuda()
    tag = f"case {case}: K={K} H={H} W={W} f={factor} parts={parts} q={q} {accum} int={integer} var={var}"
    try:
        zs = ZPartKriging(K, H, W, factor, parts, accum=accum, overlap=False, part_len=q if parts > 1 else 0)
        zc = ZPartKriging(K, H, W, factor, parts, accum=accum, overlap=True, part_len=q if parts > 1 else 0)
    except Exception as e:                             # shapes the host refuses (too few slices ...)
        print(tag, "skipped:", type(e).__name__)
        continue
    o1, v1 = zs.allocate(var)
    o2, v2 = zs.allocate(var)
    o3, v3 = zc.allocate(var)
    for o in (o1, o2, o3):
        o.fill_(float("nan"))
    try:
        zs.run(kd, o1, v1); zs.finish()
        zs.run(kd, o2, v2); zs.finish()
        zc.run(kd, o3, v3); zc.finish()
    except Exception as e:
        print(tag, "raised", type(e).__name__, str(e)[:80])
        continue
    ok = (not bool(torch.isnan(o1).any())) and torch.equal(o1, o2) and torch.equal(o1, o3)
    if var:
        ok = ok and torch.equal(v1, v2) and torch.equal(v1, v3)
    ok = ok and torch.equal(o1[::factor], kd)
    print(tag, "ok" if ok else "MISMATCH", flush=True)
    bad += (not ok)
print("mismatches:", bad)
sys.exit(1 if bad else 0)
