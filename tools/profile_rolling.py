#!/usr/bin/env python
"""Profiling helper: wall time of gpoeo_detect_rolling (Alg. 3, synchronous) on a slice of a
workload resident in HBM, next to one Alg. 1 call on the same traces."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="CFG3")
    ap.add_argument("--batch", type=int, default=2000)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2201_01684_b200 as g
    import tracegen as tg

    spec = getattr(tg, args.cfg).with_(batch=args.batch)
    p = g.params_for(spec)
    x = torch.empty((args.batch, spec.n_features * spec.n_samples), dtype=torch.float32, device="cuda")
    tg.generate_device(spec, x)
    g.detect_rolling(x, p)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = g.detect_rolling(x, p)
    t1 = time.perf_counter()
    res, _, _ = g.detect_periods(x, p)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    g.detect_periods(x, p)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(json.dumps({"cfg": args.cfg, "batch": args.batch, "rolling_s": t1 - t0, "alg1_s": t3 - t2,
                      "rolling_traces_per_s": args.batch / (t1 - t0), "mean_n_sub": float(r["n_sub"].mean()),
                      "stop_frac": float((r["smpdur_next_s"] < 0).mean())}))


if __name__ == "__main__":
    main()
