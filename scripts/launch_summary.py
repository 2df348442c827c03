#!/usr/bin/env python3
"""Summarise an ncu launch list (gpu__time_duration.sum per launch):
per-kernel count / total / median / max, and a per-step view."""
import collections
import csv
import sys


def load(path):
    rows, h = [], None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0].replace("bpdec::<unnamed>::", "").replace("void ", "")
                rows.append((name, float(d["Metric Value"]) / 1e3))
    return rows


if __name__ == "__main__":
    rows = load(sys.argv[1])
    d = collections.defaultdict(list)
    for n, t in rows:
        d[n].append(t)
    tot = sum(t for _, t in rows)
    print(f"{'kernel':28s} {'n':>5s} {'total_us':>10s} {'share':>6s} {'med_us':>8s} {'max_us':>8s}")
    for n, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        s = sorted(v)
        print(f"{n:28s} {len(v):5d} {sum(v):10.1f} {sum(v)/tot:6.3f} {s[len(s)//2]:8.1f} {s[-1]:8.1f}")
    print("total_us", round(tot, 1))
