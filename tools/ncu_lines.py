#!/usr/bin/env python
"""Aggregate an ncu source page (SASS) per CUDA source line (profiling helper).

    python tools/ncu_lines.py gpurun_out/bucket.ncu-rep score_bucket_kernel [lib.so] [--top 40] [--section I]

(--section I: the I-th "Kernel Name" block of the source page, for reports of several launches;
 --outer: attribute inlined helpers to the kernel-body line they were called from)

Maps each SASS offset of the kernel to its source line with `nvdisasm -g` on the cubin
extracted from the library (built with -lineinfo), then sums "Instructions Executed"
and the warp-stall samples per line.
"""
from __future__ import annotations

import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _op(ins: str) -> str:
    toks = ins.replace("{", " ").split()
    toks = [t for t in toks if not t.startswith("@")]
    return toks[0] if toks else ""


def sass_lines(lib: str, kernel_re: str, outer: bool = False) -> dict:
    """SASS offset -> (source line, opcode). outer: the kernel-body line an inlined helper was
    called from (nvdisasm -gi inlining chains), instead of the helper's own line."""
    tmp = tempfile.mkdtemp()
    subprocess.check_call(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, stdout=subprocess.DEVNULL)
    out = {}
    for f in os.listdir(tmp):
        if not f.endswith(".cubin"):
            continue
        txt = subprocess.run(["nvdisasm", "-gi" if outer else "-g", "-c", os.path.join(tmp, f)], capture_output=True,
                             text=True).stdout
        cur_fn, cur_line = None, None
        for ln in txt.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                cur_fn = m.group(1)
                continue
            m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
            if m:
                # with -gi a chain "helper line inlined at ..." ends with the outermost line: the last wins
                if not outer or "inlined at" not in ln:
                    cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;?\s*$", ln)
            if m and cur_fn and re.search(kernel_re, cur_fn):
                out.setdefault(cur_fn, {})[int(m.group(1), 16)] = (cur_line, _op(m.group(2)))
    return out


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    lib = sys.argv[3] if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else os.path.join(
        ROOT, "paper_2201_01684_b200", "libgpoeo.so")
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if "--section" in sys.argv:  # reports with several launches: the I-th "Kernel Name" block
        want = int(sys.argv[sys.argv.index("--section") + 1])
        starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
        rows = rows[starts[want]:starts[want + 1]]
    hdr = rows[1]
    ia, ie, ist = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    base = int(data[0][ia], 16)
    maps = sass_lines(lib, kre, outer="--outer" in sys.argv)
    # pick the function whose size matches the profile best
    isrc = hdr.index("Source")
    best = max(maps.values(), key=lambda m: sum(1 for r in data if m.get(int(r[ia], 16) - base, (0, ""))[1]
                                                 == _op(r[isrc])))
    best = {k: v[0] for k, v in best.items()}
    srcs = {}
    for f in set(v.split(":")[0] for v in best.values() if v):
        for d in (os.path.join(ROOT, "paper_2201_01684_b200", "csrc"), os.path.join(ROOT, "include")):
            if os.path.exists(os.path.join(d, f)):
                srcs[f] = open(os.path.join(d, f)).read().splitlines()
    inst, stall = defaultdict(float), defaultdict(float)
    for r in data:
        off = int(r[ia], 16) - base
        key = best.get(off) or "?"
        inst[key] += float(r[ie] or 0)
        stall[key] += float(r[ist] or 0)
    ti, ts = sum(inst.values()), sum(stall.values())
    print(f"kernel /{kre}/: {ti:.4g} warp instr, {ts:.0f} stall samples")
    for key in sorted(stall, key=lambda k: -stall[k])[:top]:
        f, _, n = key.partition(":")
        src = srcs.get(f, [])
        text = src[int(n) - 1].strip()[:90] if n.isdigit() and int(n) <= len(src) else ""
        print(f"{100 * inst[key] / ti:5.1f}% instr {100 * stall[key] / ts:5.1f}% stall  {key:22s} {text}")


if __name__ == "__main__":
    main()
