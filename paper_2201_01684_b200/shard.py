"""Multi-GPU plumbing (row e): trace shards and the NCCL all-gather of per-trace results.

Traces are independent (Alg. 1 keeps no cross-trace state), so the path shards with no
data-path collective: rank r owns a contiguous slice of the global trace index space and
runs the whole path on it; the only device-to-device transfer is one all-gather of the
24-byte `gpoeo_result` records (the north star's "NCCL all-gather ... to collect per-trace
periods"). Backend-agnostic (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

RESULT_BYTES = 24


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [first, first + count) of `total` traces for `rank`; shards hold
    ceil(total/world) traces except the tail (which may be empty)."""
    per = (total + world - 1) // world if world > 0 else total
    first = min(total, rank * per)
    count = max(0, min(total, first + per) - first)
    return first, count


def padded_shard(total: int, world: int) -> int:
    return (total + world - 1) // world


def gather_results(local, total: int, group=None):
    """All-gather per-trace result records (uint8 tensor [count * 24]) from every rank,
    padded to equal shards, and return the concatenation trimmed to `total` traces
    in global index order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    per = padded_shard(total, world)
    buf = torch.zeros(per * RESULT_BYTES, dtype=torch.uint8, device=local.device)
    buf[: local.numel()] = local
    out = torch.empty(world * per * RESULT_BYTES, dtype=torch.uint8, device=local.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return out[: total * RESULT_BYTES]


def chunk_ranges(first: int, count: int, max_chunk: int) -> list[tuple[int, int]]:
    """Split a shard [first, first + count) into consecutive chunks of at most max_chunk
    traces (config 4 at W = 2 and 4: a shard of 10^6/W traces exceeds one B200's HBM, so it is
    streamed through a resident buffer chunk by chunk)."""
    if max_chunk < 1:
        raise ValueError("max_chunk must be >= 1")
    out, pos, end = [], first, first + count
    while pos < end:
        n = min(max_chunk, end - pos)
        out.append((pos, n))
        pos += n
    return out


def detect_shard_chunked(fill, first: int, count: int, max_chunk: int, params, x_buf, results, workspace=None,
                         stream=None, on_chunk=None, detect=None):
    """Alg. 1 over this rank's shard in chunks through one resident input buffer.

    fill(x_view, first, n) writes the traces [first, first + n) into x_view (device
    generation, or a host copy); x_buf is a CUDA tensor [>= max_chunk][stride]; results is a
    uint8 CUDA tensor [count * 24] receiving the shard's records in global order. on_chunk(i,
    first, n, phase) is called with phase "filled" after fill and "done" after the detect call
    was enqueued (the bench times the detect calls alone with CUDA events there). detect
    defaults to gpoeo_detect_periods (the CPU tests pass a stand-in). Returns the workspace
    (reused across chunks)."""
    if detect is None:
        from . import detect_periods as detect

    for i, (f, n) in enumerate(chunk_ranges(first, count, max_chunk)):
        xv = x_buf[:n]
        fill(xv, f, n)
        if on_chunk:
            on_chunk(i, f, n, "filled")
        off = (f - first) * RESULT_BYTES
        _, _, workspace = detect(xv, params, workspace=workspace, results=results[off:off + n * RESULT_BYTES],
                                 stream=stream)
        if on_chunk:
            on_chunk(i, f, n, "done")
    return workspace


def detect_sharded(x_local, total: int, params, workspace=None, stream=None, group=None):
    """Run gpoeo_detect_periods on this rank's shard (CUDA tensor [count][stride]) and
    all-gather the results of all ranks (returns a uint8 tensor [total * 24])."""
    from . import detect_periods

    res, _, workspace = detect_periods(x_local, params, workspace=workspace, stream=stream)
    return gather_results(res, total, group), workspace
