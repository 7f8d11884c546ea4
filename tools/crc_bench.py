"""Device CRC-32 throughput (vk_crc32) on a C4-sized output volume vs the
host zlib.crc32 the reference uses (io.py:157); prints JSON."""
import json
import os
import sys
import time
import zlib

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_09523_b200.volume_io import crc32  # noqa: E402

n = 2_140_143_616                                   # C4 f32 output volume bytes
d = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
crc32(d, n)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    c = crc32(d, n)
    ts.append(time.perf_counter() - t0)
host = d[:268_435_456].cpu().numpy()
t0 = time.perf_counter()
hc = zlib.crc32(host)
th = time.perf_counter() - t0
assert hc == crc32(d[:268_435_456], 268_435_456)
print(json.dumps({"bytes": n, "device_s": min(ts), "device_GBps": n / min(ts) / 1e9,
                  "host_zlib_GBps_1core": host.size / th / 1e9, "crc": c}))
