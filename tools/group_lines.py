#!/usr/bin/env python
"""Group tools/ncu_lines.py output by source-line ranges (profiling helper).

    python tools/ncu_lines.py rep kernel --top 1000 | python tools/group_lines.py file.cu name:a-b ...
"""
import re
import sys


def main():
    fname = sys.argv[1]
    groups = []
    for g in sys.argv[2:]:
        name, _, rng = g.partition(":")
        a, _, b = rng.partition("-")
        groups.append((name, int(a), int(b)))
    acc = {}
    for ln in sys.stdin:
        m = re.match(r"\s*([\d.]+)% instr\s+([\d.]+)% stall\s+(\S+)", ln)
        if not m:
            continue
        i, s, key = float(m.group(1)), float(m.group(2)), m.group(3)
        f, _, n = key.partition(":")
        g = "other:" + f
        if f == fname and n.isdigit():
            for name, a, b in groups:
                if a <= int(n) <= b:
                    g = name
                    break
        acc.setdefault(g, [0.0, 0.0])
        acc[g][0] += i
        acc[g][1] += s
    for g, (i, s) in sorted(acc.items(), key=lambda x: -x[1][1]):
        print("%-34s %5.1f%% instr %5.1f%% stall" % (g, i, s))


if __name__ == "__main__":
    main()
