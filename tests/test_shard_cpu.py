"""Host-side logic of the particle-sharded mode on CPU (-m "not gpu"): the slice
arithmetic of the C ABI (hp_shard_range) and the per-generation exchange protocol — each
rank scores its slice, an allgather of padded chunks reassembles all N costs in order —
with world_size 2 over torch.distributed's gloo backend.  The slice costs come from the
oracle (test infrastructure); the GPU path is covered by tests/test_gpu_shard.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2005_07068_b200 as hp
import workloads as W


@pytest.mark.parametrize("n", [0, 1, 7, 64, 4096, 4097])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_range_partitions(n, world):
    seen = []
    chunk = (n + world - 1) // world
    for r in range(world):
        b, e = hp.hp.shard_range(n, r, world)
        assert 0 <= b <= e <= n and e - b <= chunk
        assert b == min(n, r * chunk)
        seen += list(range(b, e))
    assert seen == list(range(n))


def test_shard_range_rejects_bad_args():
    with pytest.raises(hp.HPError):
        hp.hp.shard_range(10, 2, 2)
    with pytest.raises(hp.HPError):
        hp.hp.shard_range(-1, 0, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1. the NCCL-id broadcast path (payload bytes arbitrary here)
        payload = bytes(np.random.default_rng(3).integers(0, 256, 128, dtype=np.uint8))
        got = hp.hp.broadcast_bytes(payload if rank == 0 else None, rank, 128)
        assert got == payload
        # 2. one generation's exchange: score my slice, allgather padded chunks
        cam = O.camera(48, 36)
        obs = O.synthesize(W.H_A, cam)
        poses = W.random_poses(17, 13)
        n = len(poses)
        b, e = hp.hp.shard_range(n, rank, world)
        chunk = (n + world - 1) // world
        mine = torch.full((chunk,), float("nan"), dtype=torch.float64)
        if e > b:
            mine[: e - b] = torch.from_numpy(O.eval_batch(poses[b:e], obs, threads=1))
        parts = [torch.empty(chunk, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, mine)
        full = torch.cat(parts)[:n].numpy()
        out[rank] = full.tolist()
    finally:
        dist.destroy_process_group()


def test_sharded_exchange_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    cam = O.camera(48, 36)
    ref = O.eval_batch(W.random_poses(17, 13), O.synthesize(W.H_A, cam), threads=1)
    for r in range(world):
        assert np.array_equal(np.array(out[r]), ref)  # bitwise: order and values preserved
