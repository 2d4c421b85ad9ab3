"""Data-parallel host logic on CPU (no GPU): world-size-2 gloo processes run
the control plane bench.py uses (NCCL-id broadcast, max-over-ranks timing,
barriers), the global batch sharding of src/dataset.cpp:82-103, and the
gradient-bucket plan of the C++ step driver."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

from paper_1903_05831_b200 import dist as dp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fake_id = bytes(range(128))
    nid = dp.share_nccl_id(dist, rank, lambda: fake_id)
    t = dp.max_over_ranks(dist, 10.0 + rank)
    dist.barrier()
    # GT / slots each rank would feed at step 3 with b = 2
    slots = dp.global_slots(3, rank, world, 2)
    from paper_1903_05831_b200 import detector as D
    p = D.preset("c4")
    gts = [D.make_gt(p, s) for s in slots]
    q.put((rank, nid == fake_id, t, slots, [g[0].tolist() for g in gts]))
    dist.destroy_process_group()


def test_gloo_world2_control_plane_and_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(r[1] for r in res)                 # every rank received rank 0's communicator id
    assert all(r[2] == 11.0 for r in res)          # max over ranks
    # union of the two ranks' shards == the single-rank global batch of b = 4
    union = res[0][3] + res[1][3]
    assert union == dp.global_slots(3, 0, 1, 4)
    from paper_1903_05831_b200 import detector as D
    p = D.preset("c4")
    single = [D.make_gt(p, s)[0].tolist() for s in union]
    assert res[0][4] + res[1][4] == single         # identical ground truth regardless of K


@pytest.mark.parametrize("world,b", [(1, 8), (2, 4), (4, 2), (8, 1)])
def test_global_batch_identity(world, b):
    """tests/test_trainer.cpp:116-126 analogue: K x b shards cover the same slots"""
    for step in (1, 2, 7):
        allslots = sorted(s for r in range(world) for s in dp.global_slots(step, r, world, b))
        assert allslots == list(range((step - 1) * 8, step * 8))


def test_bucket_plan_r50():
    """the C++ driver's bucket plan on the R50-C4 gradient layout (fp16, 25 MB)"""
    import paper_1903_05831_b200 as pkg
    lb = pkg.lib()
    # conv/fc slice sizes of R50-C4 in pack order (multiples of 8, as the driver aligns them)
    rng = np.random.default_rng(0)
    sizes = [64 * 7 * 7 * 8] + [int(s) * 8 for s in rng.integers(512, 300000, 60)]
    offs = np.cumsum([0] + sizes[:-1]).astype(np.int64)
    total = int(sum(sizes))
    cap = 25 * 1024 * 1024 // 2
    out = np.zeros(2 * (len(offs) + 1), np.int64)
    fn = lb.sdb_plan_buckets
    fn.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_void_p, C.c_int]
    nb = fn(offs.ctypes.data_as(C.c_void_p), len(offs), total, cap, out.ctypes.data_as(C.c_void_p), len(offs) + 1)
    b = out[: 2 * nb].reshape(nb, 2)
    assert b[0, 1] == total and b[-1, 0] == 0              # covers the buffer, last layers first
    assert all(b[i, 0] == b[i + 1, 1] for i in range(nb - 1))  # contiguous, descending
    assert set(b[:, 0]).issubset(set(offs.tolist()))        # boundaries at parameter starts
    assert all((hi - lo) >= cap for lo, hi in b[:-1])       # every bucket but the last reaches the cap
    assert nb == -(-total // cap) or nb == total // cap + 1 or nb <= total // cap + 1


def _syncbn_worker(rank, world, port, q):
    """one rank of the SyncBN aggregation protocol the GPU path runs (local FP64
    sums rounded to float into [sum, sumsq, count], one fp32 SUM allreduce,
    statistics from the global sums -- src/syncbn.cpp:21-57), over gloo"""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from tests.test_oracle_pins import _shards
    x, _, _, _ = _shards(world, 2, 24, 5, 7, 0, 10 * world)
    xr = x[rank].astype(np.float64)
    agg = np.concatenate([xr.sum(axis=(0, 2, 3)), (xr * xr).sum(axis=(0, 2, 3)), [xr.shape[0] * 35]])
    t = torch.from_numpy(agg.astype(np.float32))
    dist.all_reduce(t)
    a = t.numpy().astype(np.float64)
    Cc = 24
    mu = a[:Cc] / a[2 * Cc]
    var = np.maximum(a[Cc:2 * Cc] / a[2 * Cc] - mu * mu, 0.0)
    q.put((rank, t.numpy().tolist(), mu.astype(np.float32).tolist(), (1.0 / np.sqrt(var + 1e-5)).astype(np.float32).tolist()))
    dist.destroy_process_group()


def test_syncbn_protocol_gloo_world2(orc):
    """two gloo ranks agree bitwise on the all-reduced statistics buffer, and
    their global statistics equal the K = 2 restatement's (a 2-term float sum is
    order-free, so NCCL's reduction order cannot change it either)"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_syncbn_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res[0][1] == res[1][1]
    from oracle import p
    from tests.test_oracle_pins import _shards
    x, _, g, b = _shards(2, 2, 24, 5, 7, 0, 20)
    y = np.zeros_like(x)
    mean, inv = np.zeros(24, np.float32), np.zeros(24, np.float32)
    agg = np.zeros(49, np.float32)
    orc.orc_syncbn_forward_k(2, p(x), 2, 24, 5, 7, p(g), p(b), 1e-5, 0, p(y), p(mean), p(inv), p(agg))
    assert np.allclose(np.array(res[0][1], np.float32), agg, rtol=1e-6, atol=1e-5)
    assert np.allclose(np.array(res[0][2], np.float32), mean, rtol=1e-5, atol=1e-6)
    assert np.allclose(np.array(res[0][3], np.float32), inv, rtol=1e-5)


def _shard_worker(rank, world, port, q):
    """the sharded optimizer's collectives (csrc/detector.cpp)
    restated over gloo on the R50-C4 bucket plan: per bucket, reduce-scatter of
    the fp16 gradient (pre-multiplied by 1/K, the ncclAvg contract), apply_sgd
    (the reference rule, oracle restatement) on this rank's shard only, then an
    all-gather of the updated shard"""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    import oracle
    dist.init_process_group("gloo", rank=rank, world_size=world)
    buckets, total = _c4_buckets()
    rng = np.random.default_rng(7)
    w = rng.standard_normal(total).astype(np.float32)
    v = (0.1 * rng.standard_normal(total)).astype(np.float32)
    g_all = [(rng.standard_normal(total) * 64).astype(np.float16) for _ in range(world)]
    g = torch.from_numpy(g_all[rank].astype(np.float32) / world)  # premultiplied by 1/K
    orc = oracle.orc()
    for lo, hi in buckets:
        cnt = (hi - lo) // world
        out = torch.empty(cnt)
        dist.reduce_scatter(out, list(g[lo:hi].chunk(world)))
        s = lo + rank * cnt
        gs = np.ascontiguousarray(out.numpy())
        ws, vs = np.ascontiguousarray(w[s:s + cnt]), np.ascontiguousarray(v[s:s + cnt])
        orc.orc_apply_sgd(oracle.p(ws), oracle.p(vs), oracle.p(gs), cnt, 0.01, 0.9, 128.0)
        parts = [torch.empty(cnt) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(ws))
        w[lo:hi] = torch.cat(parts).numpy()
    q.put((rank, w.tobytes()))
    dist.destroy_process_group()


def _c4_buckets():
    """the 25 MB fp16 bucket plan of the R50-C4 detector, from the C ABI's planner"""
    from paper_1903_05831_b200 import detector as D
    lb = D.L()
    lb.sdb_plan_buckets.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_void_p, C.c_int]
    # conv/fc parameter sizes of R50-C4 in pack order (device layouts: stem input
    # channels padded to 8, RPN/fc outputs padded to 8), 16-byte aligned slices
    sizes = [64 * 7 * 7 * 8]
    for (nb, width, cout) in ((3, 64, 256), (4, 128, 512), (6, 256, 1024)):
        cin = {64: 64, 128: 256, 256: 512}[width]
        for b in range(nb):
            ci = cin if b == 0 else cout
            sizes += [width * ci, width * width * 9, cout * width] + ([cout * ci] if b == 0 else [])
    sizes += [512 * 1024 * 9, 16 * 512, 64 * 512]
    for b in range(3):
        ci = 1024 if b == 0 else 2048
        sizes += [512 * ci, 512 * 512 * 9, 2048 * 512] + ([2048 * ci] if b == 0 else [])
    sizes += [88 * 2048, 328 * 2048]
    offs, o = [], 0
    for s in sizes:
        offs.append(o)
        o += (s + 7) // 8 * 8
    offs = np.array(offs, np.int64)
    out = np.zeros(2 * len(offs) + 2, np.int64)
    nb = lb.sdb_plan_buckets(offs.ctypes.data, len(offs), o, 25 * 1024 * 1024 // 2, out.ctypes.data, len(offs) + 1)
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(nb)], o


def test_gloo_world2_sharded_optimizer_equals_allreduce_update():
    """world 2: reduce-scatter -> shard update -> all-gather gives, bit for bit,
    the replicated allreduce + full apply_sgd of the reference step tail
    (src/trainer.cpp:251-254) -- the buckets split evenly over the ranks"""
    import oracle
    buckets, total = _c4_buckets()
    assert buckets[-1][0] == 0 and sum(hi - lo for lo, hi in buckets) == total
    assert all((hi - lo) % 2 == 0 for lo, hi in buckets)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res[0][1] == res[1][1]  # replicas agree bitwise
    rng = np.random.default_rng(7)
    w = rng.standard_normal(total).astype(np.float32)
    v = (0.1 * rng.standard_normal(total)).astype(np.float32)
    g_all = [(rng.standard_normal(total) * 64).astype(np.float16) for _ in range(2)]
    gsum = (g_all[0].astype(np.float32) / 2 + g_all[1].astype(np.float32) / 2).astype(np.float32)
    orc = oracle.orc()
    orc.orc_apply_sgd(oracle.p(w), oracle.p(v), oracle.p(gsum), total, 0.01, 0.9, 128.0)
    assert np.frombuffer(res[0][1], np.float32).tobytes() == w.tobytes()
