"""Batch-sharded replicas over G GPUs: the host-side logic of the multi-GPU run.

The hot path partitions by batch and needs no collective: rank r owns images
[r*B, (r+1)*B) of the global batch (B per GPU, weak scaling) and regenerates them itself from the
counter-based generator, so every shard is an exact slice of one global batch. The executed plan
is chosen once (rank 0) and broadcast, so every rank runs identical kernels. The only
collective is after timing, for verification: an all_gather of per-image checksums, and rank 0
recomputes the first images of every shard and requires bit-identity (per-image computation never
depends on batch position: DW halos never cross images and the PW K order is fixed, reading R12).

Everything here takes the process group and a `run_probe(n0, n)` callable, so the same code runs
over NCCL in bench.py and over gloo on CPU in tests/test_multirank_gloo.py.
"""
from __future__ import annotations

import os
import socket
import sys

import torch


def shard(per_gpu: int, world: int, rank: int) -> tuple[int, int]:
    """First global image index and image count of this rank's shard."""
    if not (0 <= rank < world) or per_gpu < 1:
        raise ValueError(f"bad shard request: rank {rank} of {world}, {per_gpu} images per rank")
    return rank * per_gpu, per_gpu


def broadcast_plan(plan, world: int, src: int = 0):
    """Rank `src` chose the plan (measured refinement); every rank executes exactly that plan."""
    if world == 1:
        return plan
    box = [plan]
    torch.distributed.broadcast_object_list(box, src=src)
    return box[0]


def image_checksums(out: torch.Tensor, n: int) -> torch.Tensor:
    """Per-image float64 sums of an NHWC output (exact for int8; for floats a fingerprint that a
    bit-identical recomputation reproduces exactly, since the summation order is fixed)."""
    return out.detach().double().reshape(n, -1).sum(1)


def verify_shards(out: torch.Tensor, per_gpu: int, world: int, rank: int, run_probe, probe_images: int = 2):
    """All-gather every rank's per-image checksums; rank 0 recomputes the first `probe_images`
    images of every shard with run_probe(n0, n) -> output tensor and compares bit for bit."""
    ck = image_checksums(out, per_gpu)
    allck = [torch.empty_like(ck) for _ in range(world)]
    torch.distributed.all_gather(allck, ck)
    res = {"gathered_images": world * per_gpu, "checked": 0, "bit_identical": True}
    if rank == 0:
        k = min(probe_images, per_gpu)
        for r in range(world):
            n0, _ = shard(per_gpu, world, r)
            mine = image_checksums(run_probe(n0, k), k).to(allck[r].device)
            res["checked"] += k
            res["bit_identical"] &= bool(torch.equal(mine, allck[r][:k]))
    return res


def max_over_ranks(values, device, world: int):
    """Max over ranks of per-rank timings (the contract: time on the device, max over ranks)."""
    t = torch.tensor(list(values), device=device, dtype=torch.float64)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return [float(v) for v in t]


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_under_torchrun(nproc: int, argv: list[str]) -> None:
    """`bench.py --gpus N` started without a torchrun environment: re-exec this script under
    torch.distributed.run with N local ranks (one per GPU, rendezvous on 127.0.0.1). Never
    returns."""
    if nproc > torch.cuda.device_count():
        raise SystemExit(f"--gpus {nproc} requested but only {torch.cuda.device_count()} CUDA device(s) visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port())] + argv
    sys.stdout.flush()
    sys.stderr.flush()
    os.execvp(cmd[0], cmd)
