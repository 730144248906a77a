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


def _chunked_worker(rank, world, port, total, max_chunk, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = shard.shard_range(total, world, rank)
    x_buf = torch.zeros((max(1, min(max_chunk, count)), 1), dtype=torch.int64)  # trace index per row
    results = torch.zeros(count * shard.RESULT_BYTES, dtype=torch.uint8)
    seen = []

    def fill(xv, f, n):
        xv[:, 0] = torch.arange(f, f + n)

    def fake_detect(xv, params, workspace=None, results=None, stream=None):
        idx = xv[:, 0].numpy()
        results.copy_(torch.from_numpy(_fake_results(int(idx[0]), len(idx)).view(np.uint8).copy()))
        return results, None, workspace

    shard.detect_shard_chunked(fill, first, count, max_chunk, None, x_buf, results,
                               on_chunk=lambda i, f, n, ph: seen.append((i, f, n, ph)), detect=fake_detect)
    out = shard.gather_results(results, total)
    q.put((rank, first, count, seen, out.numpy().tobytes()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total,max_chunk", [(10, 3), (1000, 125), (7, 100), (9, 1)])
def test_chunked_shards_match_world1(total, max_chunk):
    """Config 4's streamed shards (row e): each rank runs its shard through one resident
    buffer in chunks of <= max_chunk traces; the all-gathered records equal the W = 1 ones."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunked_worker, args=(r, world, port, total, max_chunk, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _fake_results(0, total).view(np.uint8).tobytes()
    for _, first, count, seen, blob in got:
        assert blob == want
        chunks = [(f, n) for i, f, n, ph in seen if ph == "done"]
        assert chunks == shard.chunk_ranges(first, count, max_chunk)
        assert all(n <= max_chunk for _, n in chunks) and sum(n for _, n in chunks) == count


def test_chunk_ranges():
    assert shard.chunk_ranges(0, 10, 4) == [(0, 4), (4, 4), (8, 2)]
    assert shard.chunk_ranges(500_000, 500_000, 125_000) == [(500_000 + i * 125_000, 125_000) for i in range(4)]
    assert shard.chunk_ranges(5, 0, 3) == []
    with pytest.raises(ValueError):
        shard.chunk_ranges(0, 1, 0)
