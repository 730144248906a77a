#!/usr/bin/env python
"""Profiling helper (not part of the product path): run the full detector on a config-3
slice resident in HBM, print per-phase CUDA-event times, the work counters, the query mix
of the two scorer paths, and (debug builds with -DGPOEO_STATS) the bucketed scorer's
per-pair statistics. Used under `ncu` on the GPU box:

    python tools/profile_scorer.py --batch 2000 --repeat 2
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=2000)
    ap.add_argument("--repeat", type=int, default=2)
    ap.add_argument("--first", type=int, default=0)
    ap.add_argument("--maxit", type=int, default=32, help="CEM pass cap (timing experiments only)")
    ap.add_argument("--bounded", type=int, default=1, help="gpoeo_params.bounded_search")
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2201_01684_b200 as g
    import tracegen as tg

    spec = tg.CFG3.with_(batch=args.batch)
    p = g.params_for(spec)
    p.gmm_max_iters = args.maxit
    p.bounded_search = args.bounded
    x = torch.empty((args.batch, spec.n_features * spec.n_samples), dtype=torch.float32, device="cuda")
    tg.generate_device(spec, x, first=args.first, count=args.batch)
    ws = g.alloc_workspace(g.workspace_size(p, args.batch))
    res = torch.empty(args.batch * g.RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    lib = g.load()
    stats_fn = getattr(lib, "gpoeo_debug_stats", None)
    out = {}
    for r in range(args.repeat):
        if stats_fn is not None:
            buf = (ctypes.c_ulonglong * 24)()
            stats_fn(buf, 1)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        for e in evs:
            e.record()
        torch.cuda.synchronize()
        g.detect_periods_timed(x, p, ws, res, evs)
        torch.cuda.synchronize()
        out["phase_ms"] = {n: evs[i].elapsed_time(evs[i + 1]) for i, n in enumerate(g.PHASES)}
        if stats_fn is not None:
            buf = (ctypes.c_ulonglong * 24)()
            stats_fn(buf, 0)
            s = list(buf)
            out["stats"] = {"bucket_pairs": s[0], "bucket_passes_per_pair": s[1] / max(s[0], 1),
                            "swept_members_per_pass": s[2] / max(s[1], 1),
                            "straddle_members_per_pass": s[3] / max(s[1], 1),
                            "straddle_buckets_per_pass": s[4] / max(s[1], 1), "team_pairs": s[5],
                            "team_passes_per_pair": s[6] / max(s[5], 1), "team_warp_iterations": s[7],
                            "team_pair_passes": s[6],
                            "team_by_tau_class": {c: {"warp_iterations": s[12 + i], "pair_passes": s[16 + i],
                                                      "pairs": s[20 + i]}
                                                  for i, c in enumerate(["1", "2-4", "8-16", ">=32"])},
                            "bucket_cycles_per_pair": {k: s[8 + i] / max(s[0], 1) for i, k in
                                                       enumerate(["range_sort", "bucket_sums", "passes", "final"])}}
    out["counters"] = g.read_counters(ws, p, args.batch)
    # query mix from the per-trace detail (candidates + local ranges)
    _, det, _ = g.detect_periods(x, p, workspace=ws, detail=True)
    d = g.detail_numpy(det)
    r = g.results_numpy(res)
    N = spec.n_samples
    mix = {"small_q": 0, "big_q": 0, "small_pairs": 0, "big_pairs": 0, "small_samples": 0, "big_samples": 0}
    for i in range(args.batch):
        if r[i]["status"] != 0:
            continue
        Ls = set(int(v) for v in d[i]["cand_L"][: d[i]["n_candidates"]])
        Ls |= set(range(int(d[i]["local_lo"]), int(d[i]["local_hi"]) + 1))
        for L in Ls:
            k = "big" if L >= 513 else "small"
            mix[k + "_q"] += 1
            mix[k + "_pairs"] += N // L - 1
            mix[k + "_samples"] += (N // L - 1) * L
    out["query_mix"] = mix
    # team-path queries by team width tau = pow2ceil(ceil(L / 16)) (L < 513): queries, pairs
    taus = {}
    for i in range(args.batch):
        if r[i]["status"] != 0:
            continue
        Ls = set(int(v) for v in d[i]["cand_L"][: d[i]["n_candidates"]])
        Ls |= set(range(int(d[i]["local_lo"]), int(d[i]["local_hi"]) + 1))
        for L in Ls:
            if L >= 513:
                continue
            tau = 1
            while tau * 16 < L:
                tau <<= 1
            e = taus.setdefault(tau, [0, 0, 0])
            e[0] += 1
            e[1] += N // L - 1
            e[2] += (N // L - 1) * L
    out["team_taus"] = {str(k): {"queries": v[0], "pairs": v[1], "samples": v[2]} for k, v in sorted(taus.items())}
    hist = np.histogram([int(v) for v in r["period"] if v > 0], bins=[0, 64, 128, 256, 513, 1024, 2048, 4097])
    out["period_hist"] = {"edges": hist[1].tolist(), "counts": hist[0].tolist()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
