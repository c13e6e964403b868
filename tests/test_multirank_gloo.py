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
