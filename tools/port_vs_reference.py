"""CPU arm fidelity: time the oracle port against the live reference on the
same sub-parts (fit + fill, one core), and check the outputs are identical.
Build-container tool (needs /root/reference); writes profiles/port_vs_reference_r02.json."""
import json, os, sys, time
os.environ.setdefault("OMP_NUM_THREADS", "1"); os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np
from volkrig import kriging as K
from volkrig.model import VolumeGrid
from oracle import kriging_oracle as O
from paper_2303_09523_b200.phantoms import CONFIGS, phantom_planes

res = []
for name, parts in (("C4", (0, 16)), ("C2", (0, 3)), ("C3", (5,))):
    cfg = CONFIGS[name]
    ranges = O.subpart_ranges(cfg.n_known, cfg.n_subparts)
    for s in parts:
        b, e = ranges[s]
        ks = phantom_planes(cfg, cfg.known_z[b:e + 1])
        d, m = O.subpart_grid(ks, 0, e - b, cfg.factor)
        c, v = O.subpart_samples(d, m)
        t0 = time.perf_counter()
        mdl = K.fit_variogram((c, v))
        ref = K.fill_missing(VolumeGrid(d, m), mdl).data
        t_ref = time.perf_counter() - t0
        t0 = time.perf_counter()
        out, _, om = O.reconstruct_zpart(ks, 0, e - b, cfg.factor)
        t_port = time.perf_counter() - t0
        res.append({"config": name, "part": s, "reference_s": t_ref, "port_s": t_port,
                    "port_over_reference": t_port / t_ref, "identical": bool(np.array_equal(out, ref))})
        print(res[-1], flush=True)
out = {"what": "single-core time of fit_variogram + fill_missing per sub-part: live reference vs oracle port",
       "numpy": np.__version__, "rows": res,
       "mean_ratio": float(np.mean([r["port_over_reference"] for r in res]))}
json.dump(out, open(os.path.join(ROOT, "profiles", "port_vs_reference_r02.json"), "w"), indent=1)
print("mean port/reference", out["mean_ratio"])
