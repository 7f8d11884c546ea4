"""Per-CTA run times of the serial prediction launch (development tool; needs a
variant library built with -DVK_FT_DIAG=1, see tools/build_variant.sh)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2303_09523_b200 import ZPartKriging, _lib
from paper_2303_09523_b200.phantoms import CONFIGS, phantom_planes
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = CONFIGS[name]
ks = torch.from_numpy(phantom_planes(cfg, cfg.known_z)).cuda()
zk = ZPartKriging(cfg.n_known, cfg.height, cfg.width, cfg.factor, cfg.n_subparts, overlap=False, redraw_pairs=True)
for _ in range(3):
    zk.run(ks)
    zk.finish()
torch.cuda.synchronize()
lib = _lib.load()
n = 296
buf = np.zeros(4 * n, dtype=np.uint64)
rc = lib.vk_debug_cta_times(buf.ctypes.data_as(ctypes.c_void_p), n)
assert rc == 0, rc
b = buf.reshape(n, 4).astype(np.int64)
t0 = b[:, 2].min()
dur = (b[:, 3] - b[:, 2]) / 1e3
end = (b[:, 3] - t0) / 1e3
ntx = (cfg.width + 127) // 128
n_gaps = cfg.n_known - 1
tile = b[:, 1] // n_gaps
tx, ty = tile % ntx, tile // ntx
nty = (cfg.height + 31) // 32
print("kernel span us", end.max(), "dur min/mean/max", dur.min(), dur.mean(), dur.max())
for nm, m in (("interior", (tx > 0) & (tx < ntx - 1) & (ty > 0) & (ty < nty - 1)),
              ("left col", tx == 0), ("right col", tx == ntx - 1), ("top row", ty == 0), ("bottom row", ty == nty - 1)):
    if m.any():
        print(f"{nm:10s} n={m.sum():3d} dur mean {dur[m].mean():8.1f} min {dur[m].min():8.1f} max {dur[m].max():8.1f}")
sm = b[:, 0]
per_sm = {}
for i in range(n):
    per_sm.setdefault(int(sm[i]), []).append(end[i])
ends = np.array([max(v) for v in per_sm.values()])
print("per-SM end: min/mean/max", ends.min(), ends.mean(), ends.max(), "n_sm", len(ends))
order = np.argsort(dur)
print("slowest 12:", [(int(i), int(sm[i]), int(tx[i]), int(ty[i]), round(float(dur[i]), 1)) for i in order[-12:]])
print("fastest 12:", [(int(i), int(sm[i]), int(tx[i]), int(ty[i]), round(float(dur[i]), 1)) for i in order[:12]])
gpc = sm // 2
