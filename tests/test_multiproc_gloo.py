"""World-size-2 CPU tests (gloo) of the multi-GPU host logic: trace sharding of the
global index space and the all-gather of per-trace result records (row e)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2201_01684_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_results(first, count):
    # deterministic record per global trace index: period = 10 + idx, status = idx % 4, ...
    rec = np.zeros(count, dtype=[("period", "<i4"), ("period_s", "<f4"), ("error", "<f4"), ("status", "<i4"),
                                 ("best_candidate", "<i4"), ("n_candidates", "<i4")])
    idx = np.arange(first, first + count)
    rec["period"] = 10 + idx
    rec["period_s"] = 0.5 * idx
    rec["error"] = 1.0 / (1 + idx)
    rec["status"] = idx % 4
    rec["best_candidate"] = idx // 2
    rec["n_candidates"] = idx % 17
    return rec


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = shard.shard_range(total, world, rank)
    local = torch.from_numpy(_fake_results(first, count).view(np.uint8).copy())
    out = shard.gather_results(local, total)
    q.put((rank, first, count, out.numpy().tobytes()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [10, 7, 1, 2])
def test_shard_and_gather_world2(total):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _fake_results(0, total).view(np.uint8).tobytes()
    covered = sorted((f, c) for _, f, c, _ in got)
    assert sum(c for _, c in covered) == total
    assert covered[0][0] == 0 and all(covered[i][0] + covered[i][1] == covered[i + 1][0] for i in range(len(covered) - 1)
                                      if covered[i + 1][1] > 0)
    for _, _, _, blob in got:
        assert blob == want  # every rank holds all results in global order


def test_shard_ranges_partition():
    for total in (0, 1, 5, 100, 1_000_000):
        for world in (1, 2, 3, 4, 8):
            spans = [shard.shard_range(total, world, r) for r in range(world)]
            assert sum(c for _, c in spans) == total
            pos = 0
            for f, c in spans:
                if c:
                    assert f == pos
                    pos += c
            assert max(c for _, c in spans) <= shard.padded_shard(total, world) or total == 0
