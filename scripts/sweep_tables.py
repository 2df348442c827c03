#!/usr/bin/env python3
"""Markdown tables of DESIGN.md section 7 from the ET sweep JSONs.

usage: python scripts/sweep_tables.py profiles/r2/et_sweep_cfg2.json [profiles/r2/et_sweep_cfg5.json]
       python scripts/sweep_tables.py --met profiles/r2/et_sweep_met.json
"""
import json
import sys


def e(x):
    return f"{x:.2e}"


def base_table(paths):
    print("| β | D̄ PCE | D̄ VNR | FER none / PCE / VNR | edge-updates/s none / PCE / VNR | iteration gain VNR vs PCE | frames/s gain |")
    print("|---|---|---|---|---|---|---|")
    for p in paths:
        d = json.load(open(p))
        for r in d["rows"]:
            none = r.get("none")
            lab = (f"{r['beta']:.2f}" if isinstance(r.get("beta"), float)
                   else f"{d['workload']} stream, β_f ~ U{r.get('beta_range', r.get('beta'))} ({r['frames']} frames)")
            fer = " / ".join(("–" if x is None else f"{x['fer']:.3g}") for x in (none, r["pce"], r["vnr"]))
            eu = " / ".join(("–" if x is None else e(x["edge_updates_per_s"])) for x in (none, r["pce"], r["vnr"]))
            print(f"| {lab} | {r['pce']['d_bar']:.1f} | {r['vnr']['d_bar']:.1f} | {fer} | {eu} | "
                  f"{r['iteration_gain']:.1f} | {r['frame_throughput_gain']:.1f} |")


def met_table(path):
    d = json.load(open(path))
    print("| β | D̄ 250 / 500 / 1000 / VNR | FER 250 / 500 / 1000 / VNR | decoded bits/s PCE / VNR | K_VNR/K vs 250 / 500 / 1000 | SKR_dec 500 / 1000 / VNR |")
    print("|---|---|---|---|---|---|")
    for r in d["rows"]:
        pol = {"500": r["pce"], "vnr": r["vnr"]}
        for k in ("250", "1000"):
            if "pce" + k in r:
                pol[k] = r["pce" + k]
        ks = ["250", "500", "1000", "vnr"]
        db = " / ".join(f"{pol[k]['d_bar']:.1f}" if k in pol else "–" for k in ks)
        fer = " / ".join(f"{pol[k]['fer']:.3f}" if k in pol else "–" for k in ks)
        dec = f"{e(r['pce']['decoded_info_bits_per_s'])} / {e(r['vnr']['decoded_info_bits_per_s'])}"
        kr = {"250": r.get("k_vnr_over_k_pce250"), "500": r.get("k_vnr_over_k_pce"), "1000": r.get("k_vnr_over_k_pce1000")}
        ci = r.get("k_vnr_over_k_pce_ci95")
        kk = " / ".join(("–" if kr.get(k) is None else f"{kr[k]:.2f}") for k in ("250", "500", "1000"))
        if ci:
            kk += f" (500: {ci[0]:.2f}–{ci[1]:.2f})"
        sd = " / ".join(f"{pol[k]['skr_dec_eq3']:.1f}" if k in pol else "–" for k in ("500", "1000", "vnr"))
        print(f"| {r['beta']:.3f} | {db} | {fer} | {dec} | {kk} | {sd} |")
    print("beta_opt:", json.dumps(d.get("beta_opt")))


if __name__ == "__main__":
    if sys.argv[1] == "--met":
        met_table(sys.argv[2])
    else:
        base_table(sys.argv[1:])
