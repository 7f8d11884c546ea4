"""load_stack throughput (io.py:128-143): Pillow decode of 16-bit PNG slices
on host threads + device normalisation (vk_normalize_stack), against the
reference's sequence (decode + numpy f32 conversion + normalize_stack on one
core, restated by oracle/stack_oracle.py), and the normalisation kernel alone
on a device-resident C5-sized stack (512 x 1024^2 u16) vs the HBM roofline.
Prints one JSON line."""
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch
from PIL import Image

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import stack_oracle as SO                      # noqa: E402
from paper_2303_09523_b200.stack_io import SAMPLE_U16, _normalize_dev, load_stack, parse_manifest  # noqa: E402

peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
hbm = peaks.get("hbm_gbs") or peaks.get("hbm_copy_gbs") or 6455.9

# 1) kernel alone: 1 GiB of u16 samples -> 2 GiB f32 (two reads of the samples + one write)
n = 512 * 1024 * 1024
raw = torch.randint(0, 65536, (n,), device="cuda", dtype=torch.int32).to(torch.int16)
out = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(3):
    _normalize_dev(raw, SAMPLE_U16, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    e0.record()
    _normalize_dev(raw, SAMPLE_U16, out=out)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
t_k = float(np.median(ts))
alg = n * (2 + 2 + 4)
del raw, out

# 2) whole load_stack from 1024^2 16-bit PNGs
n_sl = int(os.environ.get("STACK_SLICES", "64"))
r = np.random.default_rng(0)
with tempfile.TemporaryDirectory() as d:
    base = (r.random((1024, 1024)) * 4000).astype(np.uint16)
    lines = ["pixel_spacing_mm = 1 1", "slice_gap_mm = 4"]
    for i in range(n_sl):
        Image.fromarray(base + np.uint16(i)).save(os.path.join(d, f"s{i:04d}.png"))
        lines.append(f"slice = s{i:04d}.png")
    man = os.path.join(d, "m.manifest")
    open(man, "w").write("\n".join(lines) + "\n")
    load_stack(man)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = load_stack(man)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref = SO.load_samples(parse_manifest(man).slice_files)
    t_ref = time.perf_counter() - t0
    assert np.array_equal(st.slices.cpu().numpy().view(np.uint32), ref.view(np.uint32))
print(json.dumps({
    "normalize_kernel": {"samples": n, "sample": "u16", "ms": t_k * 1e3, "alg_bytes": alg,
                         "GBps": alg / t_k / 1e9, "hbm_peak_GBps": hbm, "frac": alg / t_k / 1e9 / hbm},
    "load_stack": {"slices": n_sl, "shape": [1024, 1024], "png": "16-bit grey", "s": t_dev,
                   "slices_per_s": n_sl / t_dev, "threads": min(32, os.cpu_count() or 1)},
    "reference_sequence_1core": {"s": t_ref, "slices_per_s": n_sl / t_ref},
    "bit_identical": True}))
