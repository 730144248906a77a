#!/usr/bin/env python
"""Profiling helper (not part of the product path): throughput of the spectral stage at
config 3 (10^5 x 3 x 2^16 resident in HBM): the spectral-only detector
(gpoeo_detect_major_periods, rows a1-a3 + arg-max, nothing written but 16 B per trace)
and the power-spectrum surface, timed with CUDA events on the launching stream.

    python tools/profile_spectral.py --batch 100000 --steps 5
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=100000)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    import torch

    import paper_2201_01684_b200 as g
    import tracegen as tg

    spec = tg.CFG3.with_(batch=args.batch)
    p = g.params_for(spec)
    B = args.batch
    x = torch.empty((B, spec.n_features * spec.n_samples), dtype=torch.float32, device="cuda")
    tg.generate_device(spec, x)
    ws = g.alloc_workspace(g.major_workspace_size(p, B))
    res = torch.empty(B * g.MAJOR_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        g.detect_major_periods(x, p, workspace=ws, results=res)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        g.detect_major_periods(x, p, workspace=ws, results=res)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    alg = B * (4 * spec.n_features * spec.n_samples + 16)
    r = g.major_numpy(res)
    out = {"major_ms": ms, "traces_per_s": B / ms * 1e3, "GB_per_s": alg / ms / 1e6,
           "ok_frac": float((r["status"] == 0).mean())}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
