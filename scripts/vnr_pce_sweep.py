#!/usr/bin/env python3
"""VNR-ET vs PCE-ET report: per beta, config-2 code, one batch of
64 device-generated syndrome-mode frames, D_max = 500: mean iterations, FER
with the reference's Wilson interval (channel.cpp:63-72), edge-updates/s and
info bits/s for PCE-only and VNR+PCE, and the VNR/PCE gains.

Usage: python scripts/vnr_pce_sweep.py [out.json]   (GPU required)
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2507_03509_b200 as P  # noqa: E402
from paper_2507_03509_b200.decoder import Q_ABS  # noqa: E402

BETAS = [0.10, 0.20, 0.30, 0.40, 0.50, 0.70, 0.80, 0.90, 0.92, 0.94, 0.96, 0.98, 0.99]
FRAMES = 64


def main(out_path):
    w = P.WORKLOADS["cfg2"]
    code = w.make_code()
    N, M, E = code.n_vars, code.n_checks, code.n_edges
    dec = P.BatchDecoder(code, max_slots=FRAMES)
    llr = torch.empty((FRAMES, N), dtype=torch.float32, device="cuda")
    syn = torch.empty((FRAMES, (M + 31) // 32), dtype=torch.int32, device="cuda")
    x = torch.empty((FRAMES, (N + 31) // 32), dtype=torch.int32, device="cuda")
    out = {"iterations": torch.zeros(FRAMES, dtype=torch.int32, device="cuda"),
           "reasons": torch.zeros(FRAMES, dtype=torch.uint8, device="cuda"),
           "bits": torch.zeros((FRAMES, (N + 31) // 32), dtype=torch.int32, device="cuda")}
    rows = []
    for beta in BETAS:
        snr = P.snr_for_beta(beta, code.rate())
        dec.sample_frames_device(snr, P.FRAME_SEED, 0, FRAMES, llr, syn, x)
        row = {"beta": beta, "snr": snr, "frames": FRAMES}
        for name, cfg in (("pce", P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=False, q_mode=Q_ABS)),
                          ("vnr", P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=True, q_mode=Q_ABS))):
            dec.decode_batch(llr, cfg, syndrome=syn, packed=True, out=out)  # warm
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dec.decode_batch(llr, cfg, syndrome=syn, packed=True, out=out)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            it = out["iterations"].cpu().numpy()
            rs = out["reasons"].cpu().numpy()
            ok_bits = (out["bits"] == x).all(dim=1).cpu().numpy()
            success = (rs == 0) & ok_bits
            errors = int(FRAMES - success.sum())
            lo, hi = P.wilson_interval(errors, FRAMES)
            row[name] = {"d_bar": float(it.mean()), "fer": errors / FRAMES, "fer_ci": [lo, hi],
                         "stops": {"syndrome": int((rs == 0).sum()), "vnr": int((rs == 1).sum()),
                                   "max_iter": int((rs == 2).sum())},
                         "undetected": int(((rs == 0) & ~ok_bits).sum()),
                         "seconds": dt, "edge_updates_per_s": float(it.sum()) * E / dt,
                         "decoded_info_bits_per_s": float(success.sum()) * (N - M) / dt,
                         "processed_info_bits_per_s": FRAMES * (N - M) / dt}
        row["iteration_gain"] = row["pce"]["d_bar"] / row["vnr"]["d_bar"]
        row["frame_throughput_gain"] = row["pce"]["seconds"] / row["vnr"]["seconds"]
        rows.append(row)
        print(json.dumps({"beta": beta, "d_pce": row["pce"]["d_bar"], "d_vnr": row["vnr"]["d_bar"],
                          "fer_pce": row["pce"]["fer"], "fer_vnr": row["vnr"]["fer"],
                          "eu_pce": row["pce"]["edge_updates_per_s"], "eu_vnr": row["vnr"]["edge_updates_per_s"],
                          "gain_it": row["iteration_gain"], "gain_frames": row["frame_throughput_gain"]}),
              flush=True)
    res = {"workload": w.name, "code": {"N": N, "M": M, "E": E, "rate": code.rate()}, "d_max": w.d_max,
           "q_mode": "abs", "data": "synthetic (seeded BASELINE generator, device-generated syndrome-mode frames)",
           "gpu": torch.cuda.get_device_name(0), "rows": rows}
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "vnr_pce_sweep.json"))
