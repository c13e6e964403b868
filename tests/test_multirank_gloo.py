"""Batch sharding on CPU with torch.distributed/gloo, world_size 2.

The hot path shards by batch with no collective: each rank regenerates its image slice from the
counter-based generator; the only collective (after timing, verification only) gathers per-image
checksums. Here: every rank's shard equals its slice of the global batch, and the gathered
per-image oracle outputs equal a single-process run over the global batch, bit for bit.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import network as onet


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, per_rank, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # shard of the input batch, regenerated locally from (seed, role, global image index)
    x = synth.activations(synth.SEED, "single_dwpw/input", rank * per_rank, per_rank, 14, 14, 16, "float")
    y = onet.forward("single_dwpw", "f32", rank * per_rank, per_rank)
    ck = torch.from_numpy(y.reshape(per_rank, -1).sum(1))
    xs = torch.from_numpy(x.reshape(per_rank, -1).sum(1))
    gy = [torch.empty_like(ck) for _ in range(world)]
    gx = [torch.empty_like(xs) for _ in range(world)]
    dist.all_gather(gy, ck)
    dist.all_gather(gx, xs)
    if rank == 0:
        q.put((torch.cat(gx).numpy(), torch.cat(gy).numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_batch_shards_match_global_batch():
    world, per_rank = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    gx, gy = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x_all = synth.activations(synth.SEED, "single_dwpw/input", 0, world * per_rank, 14, 14, 16, "float")
    y_all = onet.forward("single_dwpw", "f32", 0, world * per_rank)
    assert np.array_equal(gx, x_all.reshape(world * per_rank, -1).sum(1))
    assert np.array_equal(gy, y_all.reshape(world * per_rank, -1).sum(1))


def test_shard_slices_are_exact():
    a = synth.activations(7, "r", 0, 6, 4, 4, 8, "int8")
    b = synth.activations(7, "r", 2, 3, 4, 4, 8, "int8")
    assert np.array_equal(a[2:5], b)


def _replica_worker(rank, world, port, per_rank, q):
    """The replica logic bench.py runs over NCCL (paper_2404_19331_b200/replicas.py), here over
    gloo: shard, plan broadcast, max-over-ranks timing, checksum all_gather + rank-0 re-check."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_19331_b200 import replicas
    n0, n = replicas.shard(per_rank, world, rank)
    plan = replicas.broadcast_plan({"entries": ["chosen by rank 0"]} if rank == 0 else None, world)
    t = replicas.max_over_ranks([1.0 + rank, 5.0 - rank], "cpu", world)
    out = torch.from_numpy(onet.forward("single_dwpw", "s8", n0, n))
    run_probe = lambda p0, k: torch.from_numpy(onet.forward("single_dwpw", "s8", p0, k))
    ok = replicas.verify_shards(out, per_rank, world, rank, run_probe)
    # a corrupted shard must be caught
    bad = replicas.verify_shards(out + (1 if rank == 1 else 0), per_rank, world, rank, run_probe)
    if rank == 0:
        q.put((plan, t, ok, bad))
    dist.barrier()
    dist.destroy_process_group()


def test_replica_logic_over_gloo():
    world, per_rank = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replica_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    plan, t, ok, bad = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert plan == {"entries": ["chosen by rank 0"]}
    assert t == [2.0, 5.0]
    assert ok == {"gathered_images": 6, "checked": 4, "bit_identical": True}
    assert bad["bit_identical"] is False


def test_shard_rejects_bad_requests():
    import pytest
    from paper_2404_19331_b200 import replicas
    assert replicas.shard(256, 8, 7) == (1792, 256)
    with pytest.raises(ValueError):
        replicas.shard(256, 2, 2)

