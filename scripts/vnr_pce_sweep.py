#!/usr/bin/env python3
"""ET-policy report (BASELINE configs 2 and 5): per beta (or the
mixed-beta stream of config 5), device-generated syndrome-mode frames,
D_max = 500, ET in {none, PCE, VNR(+PCE)}: mean iterations, FER with the
reference's Wilson interval (channel.cpp:63-72), edge-updates/s and info
bits/s, and the VNR/PCE gains.

Usage: python scripts/vnr_pce_sweep.py [out.json] [--workload cfg2|cfg5] [--no-none]
(GPU required)
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2507_03509_b200 as P  # noqa: E402
from paper_2507_03509_b200.decoder import Q_ABS  # noqa: E402

BETAS = [0.10, 0.20, 0.30, 0.40, 0.50, 0.70, 0.80, 0.90, 0.92, 0.94, 0.96, 0.98, 0.99]


def policies(w, with_none):
    out = []
    if with_none:
        out.append(("none", P.DecodeConfig(d_max=w.d_max, use_pce=False, use_vnr=False, q_mode=Q_ABS)))
    out.append(("pce", P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=False, q_mode=Q_ABS)))
    out.append(("vnr", P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=True, q_mode=Q_ABS)))
    return out


def measure(dec, code, cfg, llr, syn, x, out, frames):
    N, M, E = code.n_vars, code.n_checks, code.n_edges
    dec.decode_batch(llr, cfg, syndrome=syn, packed=True, out=out)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dec.decode_batch(llr, cfg, syndrome=syn, packed=True, out=out)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    it = out["iterations"].cpu().numpy()
    rs = out["reasons"].cpu().numpy()
    ok_bits = (out["bits"] == x).all(dim=1).cpu().numpy()
    # a frame is decoded when its bits equal the message; without PCE the
    # reason is max_iterations even for a correct frame
    success = ok_bits if not cfg.use_pce else (rs == 0) & ok_bits
    errors = int(frames - success.sum())
    lo, hi = P.wilson_interval(errors, frames)
    return {"d_bar": float(it.mean()), "fer": errors / frames, "fer_ci": [lo, hi],
            "stops": {"syndrome": int((rs == 0).sum()), "vnr": int((rs == 1).sum()), "max_iter": int((rs == 2).sum())},
            "undetected": int(((rs == 0) & ~ok_bits).sum()),
            "seconds": dt, "edge_updates_per_s": float(it.sum()) * E / dt,
            "decoded_info_bits_per_s": float(success.sum()) * (N - M) / dt,
            "processed_info_bits_per_s": frames * (N - M) / dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out", nargs="?", default=None)
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg5"])
    ap.add_argument("--no-none", action="store_true", help="skip ET none (D_max iterations per frame)")
    args = ap.parse_args()
    w = P.WORKLOADS[args.workload]
    frames = 64 if args.workload == "cfg2" else 1024  # cfg5: one GPU's share of the 8192-frame stream
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
    points = [(b, None) for b in BETAS] if args.workload == "cfg2" else [(None, (0.92, 1.0))]
    rows = []
    for beta, brange in points:
        if brange is None:
            snr = P.snr_for_beta(beta, code.rate())
            dec.sample_frames_device(snr, P.FRAME_SEED, 0, frames, llr, syn, x)
            row = {"beta": beta, "snr": snr, "frames": frames}
        else:
            dec.sample_frames_device(0.0, P.FRAME_SEED, 0, frames, llr, syn, x, beta_range=brange)
            row = {"beta_range": list(brange), "frames": frames}
        for name, cfg in policies(w, not args.no_none):
            row[name] = measure(dec, code, cfg, llr, syn, x, out, frames)
        row["iteration_gain"] = row["pce"]["d_bar"] / row["vnr"]["d_bar"]
        row["frame_throughput_gain"] = row["pce"]["seconds"] / row["vnr"]["seconds"]
        rows.append(row)
        print(json.dumps({"point": beta if brange is None else list(brange),
                          **{f"d_{k}": row[k]["d_bar"] for k in ("none", "pce", "vnr") if k in row},
                          **{f"fer_{k}": row[k]["fer"] for k in ("none", "pce", "vnr") if k in row},
                          **{f"eu_{k}": row[k]["edge_updates_per_s"] for k in ("none", "pce", "vnr") if k in row},
                          "gain_it": row["iteration_gain"], "gain_frames": row["frame_throughput_gain"]}),
              flush=True)
    res = {"workload": w.name, "code": {"N": N, "M": M, "E": E, "rate": code.rate()}, "d_max": w.d_max,
           "q_mode": "abs", "data": "synthetic (seeded BASELINE generator, device-generated syndrome-mode frames)",
           "gpu": torch.cuda.get_device_name(0), "rows": rows}
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
