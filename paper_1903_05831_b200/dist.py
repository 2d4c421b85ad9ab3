"""Data-parallel host plumbing (control plane only).

One process per GPU (torchrun); torch.distributed carries the tiny control
messages -- the 128-byte ncclUniqueId for libsdb's own NCCL communicator,
barriers and the max-over-ranks step time.  Every byte of gradient traffic
goes through libsdb's C++ NCCL path (csrc/comm.cpp), never through here.
Mirrors the reference's run_workers/CommGroup setup (src/comm.cpp:242-245,
451-471) and its global batch sharding (src/dataset.cpp:82-103).
"""
from __future__ import annotations

import os


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def init(backend: str = "gloo"):
    """initialise the control plane (127.0.0.1 rendezvous under torchrun)"""
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend)
    return dist


def share_nccl_id(dist, rank: int, make_id) -> bytes:
    """rank 0 creates the communicator id (make_id() -> 128 bytes) and every rank receives it"""
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    nid = obj[0]
    if not isinstance(nid, (bytes, bytearray)) or len(nid) != 128:
        raise RuntimeError("bad nccl unique id")
    return bytes(nid)


def max_over_ranks(dist, value: float) -> float:
    """the slowest rank's time (the contract's max over ranks)"""
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def global_slots(step: int, rank: int, world: int, batch: int):
    """global batch slots of one rank at a 1-based step, src/dataset.cpp:94:
    (step-1)*K*b + rank*b + j -- the union over ranks is the same global batch
    for every K with equal K*b."""
    return [(step - 1) * world * batch + rank * batch + j for j in range(batch)]
