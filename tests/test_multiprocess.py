"""N>1 plumbing on CPU (gloo, world size 2): replica sharding and the
all-gather of per-replica metric rows / histograms reassemble exactly the
single-process result, and aggregate_metrics over it is order-exact."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_06948_b200 import engine as E


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fake_rows(replicas):
    rng = np.random.default_rng(7)
    rows = rng.uniform(0, 1, (replicas, 16))
    hist = rng.integers(0, 50, (replicas, 256))
    return rows, hist


def _worker(rank, world, port, replicas, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows, hist = fake_rows(replicas)
    mine = E.shard(replicas, rank, world)
    got_rows, got_hist = E.gather_rows(dist, rows[mine], hist[mine], replicas, world, "cpu")
    q.put((rank, got_rows, got_hist))
    dist.destroy_process_group()


@pytest.mark.parametrize("replicas", [1, 5, 64])
def test_gather_rows_world2(replicas):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, replicas, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rows, hist = fake_rows(replicas)
    for _, got_rows, got_hist in res:
        assert np.array_equal(got_rows, rows)
        assert np.array_equal(got_hist, hist.sum(0))


def test_shard_covers_every_replica_once():
    for world in (1, 2, 4, 8):
        allr = sorted(r for k in range(world) for r in E.shard(1024, k, world))
        assert allr == list(range(1024))


def test_aggregate_metrics_is_replica_ordered_means():
    rows, _ = fake_rows(9)
    agg = E.aggregate(rows)
    n = 9.0
    mean = 0.0
    for r in range(9):
        mean += rows[r][2] / n  # aggregate_metrics: agg.x += r.x / n in cell order
    assert agg[2] == mean
    seq = 0.0
    for r in range(9):
        seq += rows[r][0]  # counts are summed in replica order
    assert agg[0] == seq and agg[14] == rows[:, 14].max()
