#!/usr/bin/env python3
"""Source-level hot spots of one kernel in an ncu report (needs --import-source
on / -lineinfo): instructions grouped by execution count (= the loop they sit
in) with their share of executed instructions and of warp stall samples, the
opcode mix, and the instructions with the most stall samples.

usage: python scripts/ncu_hotspots.py <prof.ncu-rep> <kernel regex> > profiles/rN/<name>.md
"""
import collections
import csv
import io
import re
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--print-source", "sass"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    name = rows[0][1]
    hdr, data = rows[1], rows[2:]
    ia, isrc, iex, ismp = (hdr.index(c) for c in ("Address", "Source", "Instructions Executed", "# Samples"))
    ilsb = hdr.index("stall_long_sb")
    seen, recs = set(), []
    for r in data:
        if len(r) <= iex or r[ia] in seen:
            continue
        try:
            n, sm = int(r[iex]), int(r[ismp] or 0)
        except ValueError:
            continue
        seen.add(r[ia])
        recs.append((r[ia], r[isrc].strip(), n, sm, int(r[ilsb] or 0)))
    ti, ts = sum(r[2] for r in recs), sum(r[3] for r in recs)
    print(f"# Source-level hot spots: `{name[:90]}`\n")
    print(f"report `{rep.split('/')[-1]}`; {ti} warp instructions executed, {ts} warp stall samples\n")
    print("## by execution count (instructions of one loop nest share a count)\n")
    print("| executions per instruction | static instructions | share of executed instructions | share of stall samples |")
    print("|---|---|---|---|")
    cls = collections.defaultdict(lambda: [0, 0, 0])
    for _, _, n, sm, _ in recs:
        c = cls[n]
        c[0] += 1
        c[1] += n
        c[2] += sm
    for n, (k, i, sm) in sorted(cls.items(), key=lambda x: -x[1][2])[:10]:
        print(f"| {n} | {k} | {100 * i / ti:.1f} % | {100 * sm / ts:.1f} % |")
    print("\n## opcode mix (executed)\n")
    ops = collections.Counter()
    for _, s, n, _, _ in recs:
        m = re.match(r"(@!?U?P[0-9T]+\s+)?([A-Z0-9_]+)", s)
        ops[m.group(2) if m else "?"] += n
    print(", ".join(f"{o} {100 * n / ti:.1f} %" for o, n in ops.most_common(16)))
    print("\n## instructions with the most stall samples\n")
    print("| samples | long-scoreboard | executions | instruction |")
    print("|---|---|---|---|")
    for a, s, n, sm, l in sorted(recs, key=lambda r: -r[3])[:12]:
        print(f"| {sm} | {l} | {n} | `{s[:70]}` |")


if __name__ == "__main__":
    main()
