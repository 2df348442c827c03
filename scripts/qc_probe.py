#!/usr/bin/env python3
"""QC / protograph codes on the same kernels: a rate-0.1
multi-edge-style protograph (90 x 100 base: 75 degree-1 columns on an
identity block, 25 columns of degree 3 / 6 / 12 spread over the rows) lifted
with circulants to N ~ 2^20, decoded like config 2 (64 syndrome-mode frames,
PCE with D_max = 50 and VNR+PCE with D_max = 500); prints edge-updates/s next
to the BASELINE config-2 code.  Usage: python scripts/qc_probe.py (GPU)."""
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


def protograph(rng):
    rows, cols, n1 = 90, 100, 75
    base = np.zeros((rows, cols), dtype=np.int32)
    for j in range(n1):  # degree-1 columns: identity block on the last 75 rows
        base[rows - n1 + j, cols - n1 + j] = 1
    hi = cols - n1
    degs = [3] * 12 + [6] * 8 + [12] * 5
    for c, d in zip(range(hi), degs):
        for r in rng.choice(rows, size=d, replace=False):
            base[r, c] += 1
    return base


def rate(code, frames, cfg):
    N, M = code.n_vars, code.n_checks
    dec = P.BatchDecoder(code, max_slots=frames)
    llr = torch.empty((frames, N), dtype=torch.float32, device="cuda")
    syn = torch.empty((frames, (M + 31) // 32), dtype=torch.int32, device="cuda")
    dec.sample_frames_device(P.snr_for_beta(0.95, code.rate()), P.FRAME_SEED, 0, frames, llr, syn)
    out = {"iterations": torch.zeros(frames, dtype=torch.int32, device="cuda"),
           "reasons": torch.zeros(frames, dtype=torch.uint8, device="cuda"),
           "bits": torch.zeros((frames, (N + 31) // 32), dtype=torch.int32, device="cuda")}
    dec.decode_batch(llr, cfg, syndrome=syn, packed=True, out=out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        dec.decode_batch(llr, cfg, syndrome=syn, packed=True, out=out)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    it = int(out["iterations"].sum().item())
    dec.close()
    return {"edge_updates_per_s": it * code.n_edges / dt, "d_bar": it / frames}


def main():
    rng = np.random.default_rng(7)
    qc = P.lift_protograph(protograph(rng), 10486, 11)
    base = P.WORKLOADS["cfg2"].make_code()
    res = {}
    for name, code in (("qc_lift", qc), ("baseline_cfg2", base)):
        res[name] = {"N": code.n_vars, "M": code.n_checks, "E": code.n_edges}
        for label, cfg in (("pce_d50", P.DecodeConfig(d_max=50, use_pce=True, use_vnr=False, q_mode=Q_ABS)),
                           ("vnr", P.DecodeConfig(d_max=500, use_pce=True, use_vnr=True, q_mode=Q_ABS))):
            res[name][label] = rate(code, 64, cfg)
        print(name, json.dumps(res[name]), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "qc_probe.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
