#!/usr/bin/env python3
"""Summarise an ncu report (and optional launch-list CSV) into profiles/.

Usage: python scripts/ncu_summary.py <prof.ncu-rep> <tag> [launches.csv]
Writes profiles/<tag>_ncu.md and profiles/<tag>_ncu.json (tag may contain a
directory, e.g. r2/cfg2_stream).  Run here (no GPU needed): ncu -i reads the
report.  bench.py measures the check kernel's traffic itself (live ncu probe).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                d[w] = {"value": r[i], "unit": units[i]}
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        d["top_stalls"] = [(n, round(v, 2)) for v, n in sorted(stalls, reverse=True)[:5]]
        res.append(d)
    return res


def to_bytes(v):
    val, unit = float(v["value"]), v["unit"].lower()
    return val * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(unit, 1)


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    launches = sys.argv[3] if len(sys.argv) > 3 else None
    res = raw(rep)
    os.makedirs(os.path.dirname(os.path.join(ROOT, "profiles", f"{tag}_ncu.json")), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu.json"), "w") as f:
        json.dump(res, f, indent=1)
    lines = [f"# ncu summary `{tag}`", "", f"source report: `{os.path.basename(rep)}` (ncu --set full --clock-control none)", ""]
    lines.append("| kernel | time | DRAM R+W | DRAM GB/s (R+W / time) | issue active % | L2 hit % | regs | top stalls |")
    lines.append("|---|---|---|---|---|---|---|---|")
    for d in res:
        k = d["kernel"].split("(")[0].replace("void bpdec::<unnamed>::", "")
        t = d.get("gpu__time_duration.sum", {})
        rb = to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"])
        tv = float(t.get("value", "nan"))
        ts = tv * {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0}.get(t.get("unit", ""), float("nan"))
        lines.append(f"| `{k}` | {t.get('value')} {t.get('unit')} | {rb / 1e6:.1f} MB | "
                     f"{rb / ts / 1e9:.0f} | "
                     f"{d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', {}).get('value')} | "
                     f"{d.get('lts__t_sector_hit_rate.pct', {}).get('value')} | "
                     f"{d.get('launch__registers_per_thread', {}).get('value')} | "
                     f"{', '.join(f'{n} {v}' for n, v in d['top_stalls'][:3])} |")
    if launches and os.path.exists(launches):
        lines += ["", "## launch list (`--metrics gpu__time_duration.sum`, cold-cache, serialised)", ""]
        with open(launches) as f:
            text = f.read()
        rows = [r for r in csv.reader(io.StringIO(text[text.index('"ID"'):]))] if '"ID"' in text else []
        if rows:
            hdr = rows[0]
            ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
            agg = {}
            for r in rows[1:]:
                if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
                    continue
                k = r[ki].split("(")[0].replace("void bpdec::<unnamed>::", "")
                a = agg.setdefault(k, [0, 0.0])
                a[0] += 1
                a[1] += float(r[vi].replace(",", ""))
            tot = sum(v[1] for v in agg.values())
            lines.append("| kernel | launches | total | share |")
            lines.append("|---|---|---|---|")
            for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                lines.append(f"| `{k}` | {n} | {t:.0f} | {100 * t / tot:.1f}% |")
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
