"""CPU, world_size 2 over gloo: Z sub-part sharding with the one-slice halo
exchange and the gather to rank 0 reproduces the single-device partition
exactly.  The kriging itself is the oracle here (injected), since the device
path needs a GPU; this checks the host-side partition / exchange / merge."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_reconstruct(stack, factor, n_parts, part_len):
    import torch
    from oracle import kriging_oracle as O
    ks = stack.numpy()
    K = ks.shape[0]
    q = part_len
    depth = (K - 1) * factor + 1
    vol = np.empty((depth,) + ks.shape[1:], np.float32)
    for s in range(n_parts):
        b, e = s * q, ((s + 1) * q if s < n_parts - 1 else K - 1)
        out, _, _ = O.reconstruct_zpart(ks, b, e, factor)
        vol[b * factor:b * factor + out.shape[0]] = out
    return torch.from_numpy(vol)


def _worker(rank, world, port, ks, factor, n_parts, result_q):
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2303_09523_b200.zshard import reconstruct_sharded, strong_shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = strong_shard(ks.shape[0], n_parts, rank, world)
    owned = torch.from_numpy(ks[sh.k0:sh.k1 + 1].copy())
    vol = reconstruct_sharded(owned, factor, sh, reconstruct=_oracle_reconstruct)
    # halo received in place (bench.py: straight into the stack's trailing slot)
    from paper_2303_09523_b200.zshard import exchange_halo
    slot = torch.full((2,) + ks.shape[1:], -1.0)
    exchange_halo(owned[0].contiguous(), rank, world, out=slot[1] if rank < world - 1 else None)
    if rank < world - 1:
        assert torch.equal(slot[1], torch.from_numpy(ks[sh.k1 + 1]))   # rank + 1 owns k1 + 1 first
    if rank == 0:
        result_q.put(vol.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("K,n_parts,factor", [(9, 4, 2), (17, 4, 4), (18, 4, 2)])
def test_sharded_equals_single(K, n_parts, factor):
    from oracle import kriging_oracle as O
    from paper_2303_09523_b200.phantoms import known_slices, small_config
    from paper_2303_09523_b200.zshard import check_cover, strong_shard
    cfg = small_config("head", 24, 28, K, factor, n_subparts=n_parts, seed=5)
    ks = known_slices(cfg)
    world = 2
    check_cover([strong_shard(K, n_parts, r, world) for r in range(world)], K)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ks, factor, n_parts, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref, _, _ = O.reconstruct_zparts(ks, factor, n_parts)
    assert np.array_equal(got, ref)
