#!/usr/bin/env python
"""Write profiles/ncu_traffic.json from two ncu CSV launch lists (profiling helper):

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file A.csv \\
        python tools/profile_scorer.py --batch B --repeat 1
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file S.csv \\
        python tools/profile_spectral.py --batch B --steps 1 --warmup 0
    python tools/ncu_traffic.py A.csv S.csv B [OUT.json]   (default profiles/ncu_traffic.json)

DRAM bytes (read + write) per trace of the Alg. 2 scorer kernels (every score_* launch of
the first detect call) and of the spectral-only fused kernel.
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = list(csv.reader(open(path)))
    h = None
    out = defaultdict(float)  # launch ID -> bytes
    names = {}
    for r in rows:
        if r and r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            i = int(r[h.index("ID")])
            names[i] = r[h.index("Kernel Name")]
            unit = r[h.index("Metric Unit")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            out[i] += float(r[h.index("Metric Value")].replace(",", "")) * scale
    return [(names[i], out[i]) for i in sorted(out)]


def main():
    a, sp, B = sys.argv[1], sys.argv[2], int(sys.argv[3])
    la = launches(a)
    # the first detect call: launches up to and including the first final_kernel
    first = []
    for n, b in la:
        first.append((n, b))
        if "final_kernel" in n:
            break
    scorer = sum(b for n, b in first if "score_" in n)
    ls = [b for n, b in launches(sp) if "fused_spectrum" in n]
    out = {
        "scorer_dram_bytes_per_trace": scorer / B,
        "spectral_only_dram_bytes_per_trace": ls[0] / B if ls else None,
        "note": f"ncu dram__bytes_read.sum + dram__bytes_write.sum, config-3 slice of {B} traces: all score_* "
                "launches of one detect call (candidate + local phases) per trace; fused spectral kernel in "
                "spectral-only mode per trace (algorithmic 786448 B)",
        "launches": [{"kernel": n[:80], "dram_bytes": b} for n, b in first],
    }
    path = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "profiles", "ncu_traffic.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "launches"}))


if __name__ == "__main__":
    main()
