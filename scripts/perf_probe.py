#!/usr/bin/env python3
"""Kernel-level performance probe on one GPU (development tool).

Times steady-state iterations (PCE, fixed D_max) and the VNR batch for a few
slot counts, and prints per-kernel time shares and model-A / model-B
bandwidths.  Usage: python scripts/perf_probe.py [workload] [frames]
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


def model_b_bytes(code):
    deg = code.var_degrees()
    ptr, var = code.csr()
    n1 = int((deg == 1).sum())
    nv = int((deg >= 2).sum())
    eh = int(np.isin(var, np.nonzero(deg >= 2)[0]).sum()) if code.n_edges < 10_000_000 else None
    # check pass: c2v R+W on hi edges + llr of degree-1 vars (+ post gathers from L2)
    # var pass: c2v R on hi edges + llr_h R + post W
    return {"check": 8 * eh + 4 * n1, "var": 4 * eh + 8 * nv, "eh": eh, "n1": n1, "nv": nv}


def run(wname="cfg2", frames=64):
    w = P.WORKLOADS[wname]
    code = w.make_code()
    mb = model_b_bytes(code)
    E = code.n_edges
    snr = P.snr_for_beta(0.95, code.rate())
    N, M = code.n_vars, code.n_checks
    d_llr = torch.empty((frames, N), dtype=torch.float32, device="cuda")
    d_syn = torch.empty((frames, (M + 31) // 32), dtype=torch.int32, device="cuda")
    res = {"workload": w.name, "E": E, **{k: v for k, v in mb.items()}}
    for slots in (frames, max(32, frames // 2)):
        dec = P.BatchDecoder(code, max_slots=slots)
        dec.sample_frames_device(snr, P.FRAME_SEED, 0, frames, d_llr, d_syn)
        out = {"iterations": torch.zeros(frames, dtype=torch.int32, device="cuda"),
               "reasons": torch.zeros(frames, dtype=torch.uint8, device="cuda"),
               "bits": torch.zeros((frames, (N + 31) // 32), dtype=torch.int32, device="cuda")}
        for label, cfg in (("pce_d50", P.DecodeConfig(d_max=50, use_pce=True, use_vnr=False, q_mode=Q_ABS)),
                           ("vnr", P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=True, q_mode=Q_ABS))):
            if label == "pce_d50" and slots != frames:
                continue
            dec.decode_batch(d_llr, cfg, syndrome=d_syn, packed=True, out=out)  # warm
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reps = 3
            for _ in range(reps):
                dec.decode_batch(d_llr, cfg, syndrome=d_syn, packed=True, out=out)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / reps
            it = int(out["iterations"].sum().item())
            dec.reset_profile()
            dec.set_profiling(True)
            dec.decode_batch(d_llr, cfg, syndrome=d_syn, packed=True, out=out)
            prof = dec.profile()
            dec.set_profiling(False)
            fi = prof["frame_iterations"]
            kms = {k: prof[k]["ms"] for k in dec.KERNELS}
            r = {"slots": slots, "wall_ms": dt * 1e3, "iters": it, "eu_per_s": it * E / dt,
                 "kernel_ms": kms, "frame_iters": fi,
                 "check_modelA_GBs": 8 * E * fi / (kms["check"] / 1e3) / 1e9,
                 "check_modelB_GBs": mb["check"] * fi / (kms["check"] / 1e3) / 1e9,
                 "var_modelB_GBs": mb["var"] * fi / (kms["variable"] / 1e3) / 1e9,
                 "iter_modelA_GBs": (16 * E + 4 * N + (N + M) / 8) * fi / (sum(kms.values()) / 1e3) / 1e9}
            res[f"{label}_s{slots}"] = r
            print(label, json.dumps(r), flush=True)
        dec.close()
    return res


if __name__ == "__main__":
    wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    fr = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    res = run(wl, fr)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"probe_{wl}_{fr}.json"), "w") as f:
        json.dump(res, f, indent=1)
