"""HBM probe: write-only (fill), read-only (sum), copy bandwidth on one GPU
with CUDA events (best of N) -- context for the streaming kernel's roofline,
which moves 88% writes."""
import json
import torch

n = 1 << 29                                  # 2 GiB of f32
x = torch.empty(n, dtype=torch.float32, device="cuda")
y = torch.empty_like(x)
x.fill_(1.0)


def best(fn, reps=10):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    t = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    return min(t)


b = n * 4
res = {"fill_write_gbs": b / best(lambda: x.fill_(2.0)) / 1e6,
       "sum_read_gbs": b / best(lambda: x.sum()) / 1e6,
       "copy_rw_gbs": 2 * b / best(lambda: y.copy_(x)) / 1e6}
print(json.dumps(res))
