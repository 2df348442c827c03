#!/usr/bin/env python3
"""ET-policy report (BASELINE configs 2 and 5): per beta (or the
mixed-beta stream of config 5), device-generated syndrome-mode frames,
D_max = 500, ET in {none, PCE, VNR(+PCE)}: mean iterations, FER with the
reference's Wilson interval (channel.cpp:63-72), edge-updates/s and info
bits/s, and the VNR/PCE gains.

For codes whose FER falls below 1 (--workload met): decoded info bits/s per
policy and the decoder throughput ratio of Eq. (2),
K_VNR / K = (D_bar_Dmax / D_bar_VNR) * (1 - FER_VNR) / (1 - FER_Dmax), for
D_max in --dmax (PCE-ET in both, as in the paper's simulations).

Usage: python scripts/vnr_pce_sweep.py [out.json] [--workload W] [--betas ...]
       [--frames F] [--batches B] [--dmax 250 500] [--no-none]
(GPU required)
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2507_03509_b200 as P  # noqa: E402
from paper_2507_03509_b200 import qkd  # noqa: E402
from paper_2507_03509_b200.decoder import Q_ABS  # noqa: E402

BETAS = [0.10, 0.20, 0.30, 0.40, 0.50, 0.70, 0.80, 0.90, 0.92, 0.94, 0.96, 0.98, 0.99]


def policies(w, with_none, dmaxes):
    out = []
    if with_none:
        out.append(("none", P.DecodeConfig(d_max=w.d_max, use_pce=False, use_vnr=False, q_mode=Q_ABS)))
    out.append(("pce", P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=False, q_mode=Q_ABS)))
    for d in dmaxes:
        if d != w.d_max:
            out.append((f"pce{d}", P.DecodeConfig(d_max=d, use_pce=True, use_vnr=False, q_mode=Q_ABS)))
    out.append(("vnr", P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=True, q_mode=Q_ABS)))
    return out


class Acc:
    """Per-policy totals over the batches of one beta point."""

    def __init__(self):
        self.frames = self.errors = self.success = self.undetected = self.iters = 0
        self.seconds = 0.0
        self.stops = [0, 0, 0]
        self.per_frame_it = []   # per-frame iterations / success, for the paired bootstrap of Eq. (2) ratios
        self.per_frame_ok = []

    def add(self, cfg, out, x, dt):
        it = out["iterations"].cpu().numpy()
        rs = out["reasons"].cpu().numpy()
        ok_bits = (out["bits"] == x).all(dim=1).cpu().numpy()
        # a frame is decoded when its bits equal the message; without PCE the
        # reason is max_iterations even for a correct frame
        success = ok_bits if not cfg.use_pce else (rs == 0) & ok_bits
        self.frames += len(it)
        self.success += int(success.sum())
        self.errors += int(len(it) - success.sum())
        self.undetected += int(((rs == 0) & ~ok_bits).sum())
        self.iters += int(it.sum())
        self.per_frame_it.append(it.astype(np.int64))
        self.per_frame_ok.append(success.astype(np.int64))
        self.seconds += dt
        for k in range(3):
            self.stops[k] += int((rs == k).sum())

    def row(self, code):
        N, M, E = code.n_vars, code.n_checks, code.n_edges
        lo, hi = P.wilson_interval(self.errors, self.frames)
        return {"frames": self.frames, "d_bar": self.iters / self.frames, "fer": self.errors / self.frames,
                "fer_ci": [lo, hi],
                "stops": {"syndrome": self.stops[0], "vnr": self.stops[1], "max_iter": self.stops[2]},
                "undetected": self.undetected, "seconds": self.seconds,
                "edge_updates_per_s": self.iters * E / self.seconds,
                "decoded_info_bits_per_s": self.success * (N - M) / self.seconds,
                "processed_info_bits_per_s": self.frames * (N - M) / self.seconds}


def k_ratio_ci(a_vnr, a_pce, n_boot=2000, seed=1):
    """95 % interval of K_VNR / K_PCE (Eq. 2: K ~ (1 - FER) / D_bar) by a
    paired bootstrap over frames: both policies decoded the same frames
    (common random numbers), so frames are resampled jointly."""
    iv, ov = np.concatenate(a_vnr.per_frame_it), np.concatenate(a_vnr.per_frame_ok)
    ip, op = np.concatenate(a_pce.per_frame_it), np.concatenate(a_pce.per_frame_ok)
    n = len(iv)
    rng = np.random.default_rng(seed)
    vals = []
    for _ in range(n_boot):
        idx = rng.integers(0, n, n)
        sv, sp = ov[idx].sum(), op[idx].sum()
        if sp == 0 or sv == 0:
            continue
        vals.append((ip[idx].sum() / iv[idx].sum()) * (sv / sp))
    if len(vals) < n_boot // 2:
        return None
    return [float(np.percentile(vals, 2.5)), float(np.percentile(vals, 97.5))]


def timed_decode(dec, cfg, llr, syn, out):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dec.decode_batch(llr, cfg, syndrome=syn, packed=True, out=out)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out", nargs="?", default=None)
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--betas", type=float, nargs="*", default=None)
    ap.add_argument("--frames", type=int, default=None, help="frames per batch")
    ap.add_argument("--batches", type=int, default=1, help="batches per beta point (frames for the FER CI)")
    ap.add_argument("--dmax", type=int, nargs="*", default=[], help="extra PCE-only D_max values (Eq. 2 ratios)")
    ap.add_argument("--no-none", action="store_true", help="skip ET none (D_max iterations per frame)")
    args = ap.parse_args()
    w = P.WORKLOADS[args.workload]
    mixed = args.workload == "cfg5"
    frames = args.frames or (1024 if mixed else 64)  # cfg5: one GPU's share of the 8192-frame stream
    out_path = args.out or os.path.join(ROOT, "gpurun_out", f"et_sweep_{args.workload}.json")
    code = w.make_code()
    N, M, E = code.n_vars, code.n_checks, code.n_edges
    dec = P.BatchDecoder(code, max_slots=frames)
    llr = torch.empty((frames, N), dtype=torch.float32, device="cuda")
    syn = torch.empty((frames, (M + 31) // 32), dtype=torch.int32, device="cuda")
    x = torch.empty((frames, (N + 31) // 32), dtype=torch.int32, device="cuda")
    out = {"iterations": torch.zeros(frames, dtype=torch.int32, device="cuda"),
           "reasons": torch.zeros(frames, dtype=torch.uint8, device="cuda"),
           "bits": torch.zeros((frames, (N + 31) // 32), dtype=torch.int32, device="cuda")}
    betas = args.betas if args.betas else (BETAS if args.workload == "cfg2" else list(w.betas))
    points = [(None, (0.92, 1.0))] if mixed else [(b, None) for b in betas]
    pols = policies(w, not args.no_none, args.dmax)
    rows = []
    warmed = False
    for beta, brange in points:
        acc = {name: Acc() for name, _ in pols}
        for bi in range(args.batches):
            first = bi * frames
            if brange is None:
                snr = P.snr_for_beta(beta, code.rate())
                dec.sample_frames_device(snr, P.FRAME_SEED, first, frames, llr, syn, x)
            else:
                dec.sample_frames_device(0.0, P.FRAME_SEED, first, frames, llr, syn, x, beta_range=brange)
            for name, cfg in pols:
                if not warmed:
                    timed_decode(dec, cfg, llr, syn, out)
                    warmed = True
                acc[name].add(cfg, out, x, timed_decode(dec, cfg, llr, syn, out))
        row = {"beta": beta, "frames": frames * args.batches} if brange is None else \
            {"beta_range": list(brange), "frames": frames * args.batches}
        if brange is None:
            row["snr"] = P.snr_for_beta(beta, code.rate())
        for name, _ in pols:
            row[name] = acc[name].row(code)
        row["iteration_gain"] = row["pce"]["d_bar"] / row["vnr"]["d_bar"]
        row["frame_throughput_gain"] = row["pce"]["seconds"] / row["vnr"]["seconds"]
        # Eq. (2): K = N R (1 - FER) / D_bar per iteration latency
        for name, _ in pols:
            if name.startswith("pce") and row[name]["fer"] < 1.0:
                row[f"k_vnr_over_k_{name}"] = (row[name]["d_bar"] / row["vnr"]["d_bar"]) * \
                    (1.0 - row["vnr"]["fer"]) / (1.0 - row[name]["fer"])
                row[f"k_vnr_over_k_{name}_ci95"] = k_ratio_ci(acc["vnr"], acc[name])
        # Eq. (1)-(3) at the paper's operating point (V_A such that I_AB =
        # R / beta; 80 km, eta 0.4, nu_el 0.01, xi 0.001, heterodyne,
        # N_privacy 1e8): SKR per pulse, K and SKR_dec per iteration latency,
        # and SKR_dec in bits/s with the measured decode time
        if brange is None:
            for name, _ in pols:
                r = row[name]
                b = qkd.evaluate(code.rate(), beta, r["fer"], N, max(r["d_bar"], 1.0))
                r["skr_bits_per_pulse"] = b.skr
                r["k_eq2"] = b.k_throughput
                r["skr_dec_eq3"] = b.skr_dec
                r["skr_dec_bits_per_s"] = b.skr * (r["frames"] * N / 2.0) / r["seconds"]
                r["skr_negative"] = b.negative
        rows.append(row)
        print(json.dumps({"point": beta if brange is None else list(brange),
                          **{f"d_{k}": row[k]["d_bar"] for k, _ in pols},
                          **{f"fer_{k}": row[k]["fer"] for k, _ in pols},
                          **{f"dec_bits_{k}": row[k]["decoded_info_bits_per_s"] for k, _ in pols},
                          **{k: v for k, v in row.items() if k.startswith("k_vnr")},
                          "gain_it": row["iteration_gain"], "gain_frames": row["frame_throughput_gain"]}),
              flush=True)
    beta_opt = {}
    if not mixed:
        for name, _ in pols:
            recs = [qkd.SweepRecord(r["beta"], r[name]["skr_bits_per_pulse"], r[name]["skr_dec_eq3"]) for r in rows]
            bs, bd = qkd.optimize_beta(recs)
            beta_opt[name] = {"skr": bs, "skr_dec": bd}
        print(json.dumps({"beta_opt": beta_opt}), flush=True)
    res = {"workload": w.name, "beta_opt": beta_opt,
           "qkd_params": "paper simulation point: 80 km, 0.2 dB/km, eta 0.4, nu_el 0.01, xi 0.001, heterodyne, "
                         "N_privacy 1e8, V_A such that I_AB = R / beta (paper_2507_03509_b200/qkd.py)", "code": {"N": N, "M": M, "E": E, "rate": code.rate()}, "d_max": w.d_max,
           "q_mode": "abs", "data": "synthetic (seeded generator, device-generated syndrome-mode frames)",
           "gpu": torch.cuda.get_device_name(0), "rows": rows}
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
