"""PCIe / host-copy probe for the end-to-end leg (C4 shapes): pinned D2H of
the whole output volume, D2H of only the interpolated planes (strided 2D
copy), H2D of the known slices, and a strided host-to-host copy of the known
slices into the output volume, alone and overlapped.  Prints JSON."""
import ctypes
import json
import time

import torch

cudart = ctypes.CDLL("libcudart.so")
cudart.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                     ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
H = W = 512
K, f = 256, 8
T = (K - 1) * f + 1
plane = H * W * 4
dev_out = torch.empty((T, H, W), device="cuda")
dev_in = torch.empty((K, H, W), device="cuda")
host_out = torch.empty((T, H, W)).pin_memory()
host_in = torch.empty((K, H, W)).pin_memory()


def timed(fn, n=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts)


s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def d2h_full(s=None):
    with torch.cuda.stream(s or torch.cuda.current_stream()):
        host_out.copy_(dev_out, non_blocking=True)


def d2h_missing(s=None):
    s = s or torch.cuda.current_stream()
    # gaps: planes k*f+1 .. k*f+f-1 for k < K-1: width (f-1) planes, pitch f planes
    r = cudart.cudaMemcpy2DAsync(ctypes.c_void_p(host_out.data_ptr() + plane), f * plane,
                                 ctypes.c_void_p(dev_out.data_ptr() + plane), f * plane,
                                 (f - 1) * plane, K - 1, 2, ctypes.c_void_p(s.cuda_stream))
    assert r == 0, r


def h2h_known(s=None):
    s = s or torch.cuda.current_stream()
    r = cudart.cudaMemcpy2DAsync(ctypes.c_void_p(host_out.data_ptr()), f * plane,
                                 ctypes.c_void_p(host_in.data_ptr()), plane, plane, K, 0,
                                 ctypes.c_void_p(s.cuda_stream))
    assert r == 0, r


def h2d(s=None):
    with torch.cuda.stream(s or torch.cuda.current_stream()):
        dev_in.copy_(host_in, non_blocking=True)


def all_overlapped():
    d2h_missing(s1)
    h2h_known(s2)
    h2d(s3)


res = {}
for name, fn, nbytes in (("d2h_full", d2h_full, T * plane), ("d2h_missing_2d", d2h_missing, (K - 1) * (f - 1) * plane),
                         ("h2h_known_2d", h2h_known, K * plane), ("h2d_known", h2d, K * plane),
                         ("overlapped_d2h_missing+h2h+h2d", all_overlapped, None)):
    t = timed(fn)
    res[name] = {"ms": t * 1e3, "GBps": (nbytes / t / 1e9) if nbytes else None}
print(json.dumps(res))

# the library's download (vk_plan_download) on the same shapes
import os, sys  # noqa: E401,E402
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_09523_b200 import ZPartKriging  # noqa: E402
zk = ZPartKriging(K, H, W, f, 32)
res2 = {}
for name, fn in (("download", lambda: zk.download(dev_out, host_in, host_out)),
                 ("download+h2d", lambda: (zk.download(dev_out, host_in, host_out, stream=s1), h2d(s3))),
                 ("full_d2h+h2d", lambda: (d2h_full(s1), h2d(s3)))):
    res2[name] = {"ms": timed(fn) * 1e3}
print(json.dumps(res2))
