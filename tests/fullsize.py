"""Test helpers for the full-size BASELINE configs: parallel phantom generation
(each plane is seeded independently, so any split is bit-identical to the
serial generator) and the CPU oracle's per-part fill run on a process pool.
Test infrastructure only."""

from __future__ import annotations

import hashlib
import json
import multiprocessing
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def golden_fits() -> dict:
    return json.load(open(os.path.join(HERE, "golden", "reference_fits.json")))


def _planes(args):
    from paper_2303_09523_b200.phantoms import CONFIGS, phantom_planes
    name, zs = args
    return phantom_planes(CONFIGS[name], zs)


def _workers() -> int:
    return max(1, min(32, len(os.sched_getaffinity(0))))


def known_slices(name: str) -> np.ndarray:
    from paper_2303_09523_b200.phantoms import CONFIGS
    cfg = CONFIGS[name]
    zs = cfg.known_z
    n = _workers()
    if n == 1 or len(zs) < 32:
        from paper_2303_09523_b200.phantoms import known_slices as ks
        return ks(cfg)
    chunks = [zs[i::n] for i in range(n)]
    out = np.empty((len(zs), cfg.height, cfg.width), np.float32)
    with ProcessPoolExecutor(n, mp_context=multiprocessing.get_context("spawn")) as ex:
        for i, planes in enumerate(ex.map(_planes, [(name, c) for c in chunks])):
            out[i::n] = planes
    return out


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _fill_part(args):
    from oracle import kriging_oracle as O
    path, b, e, factor, model, drift = args
    ks = np.load(path, mmap_mode="r")
    data, mask = O.subpart_grid(np.asarray(ks[b:e + 1]), 0, e - b, factor)
    out, _ = O.fill_missing(data, mask, O.Model("exponential", *model), drift)
    return out


def oracle_parts(ks: np.ndarray, factor: int, ranges, models, drift="linear", tmpdir="/tmp"):
    """Oracle fill of every Z sub-part (its grid with the trailing halo plane)
    with the given per-part models ((nugget, sill, range) tuples), on a
    process pool; yields (part, b, e, filled grid) in part order."""
    path = os.path.join(tmpdir, f"vk_known_{os.getpid()}.npy")
    np.save(path, ks)
    try:
        jobs = [(path, b, e, factor, tuple(models[s]), drift) for s, (b, e) in enumerate(ranges)]
        with ProcessPoolExecutor(_workers(), mp_context=multiprocessing.get_context("spawn")) as ex:
            for s, ((b, e), out) in enumerate(zip(ranges, ex.map(_fill_part, jobs))):
                yield s, b, e, out
    finally:
        os.unlink(path)
