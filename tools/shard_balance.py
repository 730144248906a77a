#!/usr/bin/env python
"""Profiling helper: shard-to-shard work imbalance of config 4 (8 contiguous shards of S traces,
each timed with CUDA events on one GPU): python tools/shard_balance.py 12500"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_01684_b200 as g  # noqa: E402
import tracegen as tg  # noqa: E402
spec = tg.CFG4
W, S = 8, int(sys.argv[1]) if len(sys.argv) > 1 else 12500
p = g.params_for(spec)
x = torch.empty((S, spec.n_features * spec.n_samples), dtype=torch.float32, device="cuda")
ws = g.alloc_workspace(g.workspace_size(p, S))
times = []
for r in range(W):
    first = r * (spec.batch // W)
    tg.generate_device(spec, x, first=first, count=S)
    g.detect_periods(x, p, workspace=ws); torch.cuda.synchronize()
    ts = []
    for rep in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.detect_periods(x, p, workspace=ws); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    times.append(min(ts))
t = np.array(times)
print(json.dumps({"shard_traces": S, "shards": W, "ms": [round(v, 1) for v in times], "max_over_mean": float(t.max() / t.mean())}))
