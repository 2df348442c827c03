#!/usr/bin/env python3
"""Regenerates the golden fixtures from the COMPILED REFERENCE (oracle/_ref,
built from /root/reference by `make -C oracle`).  Run in the build container:

    python tests/golden/make_golden.py

Outputs (committed):
  kat.json              known-answer values as computed by
                        the reference itself
  cfg1_reference.npz    BASELINE config-1 code, 8 seeded frames, reference
                        outputs for ET none / PCE / VNR(+PCE) in the
                        all-zero-equivalent form, plus the one-ulp tie masks
  lift36_reference.npz  the reference's (3,6) lift, 8 frames at beta 0.7
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import paper_2507_03509_b200 as P  # noqa: E402
from _parity import ref_ties  # noqa: E402

MODES = {"none": (False, False), "pce": (True, False), "vnr": (True, True)}


def kats(R):
    out = {}
    spc = R.code_from_csr(3, 1, [0, 3], [0, 1, 2])
    r = spc.decode_batch(np.array([[2.0, 2.0, -0.5]]), d_max=1, use_pce=False)
    out["spc_posteriors"] = r["posteriors"][0].tolist()
    out["spc_bits"] = r["bits"][0].tolist()
    out["spc_reason"] = int(r["reasons"][0])
    r = spc.decode_batch(np.array([[50.0, 50.0, 50.0]]))
    out["noiseless_iterations"] = int(r["iterations"][0])
    out["noiseless_reason"] = int(r["reasons"][0])
    d1 = R.code_from_csr(2, 1, [0, 1], [0])
    r = d1.decode_batch(np.array([[-1.0, 3.0]]), d_max=1, use_pce=False)
    out["deg1_posteriors"] = r["posteriors"][0].tolist()
    sat = R.code_from_csr(4, 1, [0, 3], [0, 1, 2])
    for name, l in (("sat_30_30", [30.0, 30.0, 0.0, 1.0]), ("sat_12_14", [12.0, 14.0, 0.0, 1.0]),
                    ("sat_20_25", [20.0, 25.0, 0.0, 1.0])):
        out[name] = float(sat.decode_batch(np.array([l]), d_max=1, use_pce=False)["posteriors"][0][2])
    out["snr_for_beta"] = {f"{b},{r_}": R.snr_for_beta(b, r_) for b, r_ in ((1.0, 0.02), (0.95, 0.1), (0.98, 0.02),
                                                                         (0.5, 0.25))}
    out["noise_7_0"] = R.noise_normal(7, 0, 4).tolist()
    lift = R.lift_protograph([[3, 3]], 1024, 1)
    out["lift36_dims"] = [lift.n_vars, lift.n_checks, lift.n_edges]
    obs = spc.decode_observed(np.array([0.3, -0.2, 0.1]), d_max=5, use_pce=False, use_vnr=False)
    out["observer_calls_pce_off"] = obs["calls"]
    return out


def frames_reference(R, code, llr_eq, d_max, name):
    ptr, var = code.csr()
    rc = R.code_from_csr(code.n_vars, code.n_checks, ptr, var)
    z = {"llr_eq": llr_eq.astype(np.float32), "d_max": np.int32(d_max), "check_ptr": ptr, "check_vars": var,
         "n_vars": np.int32(code.n_vars)}
    for mode, (pce, vnr) in MODES.items():
        a, tie = ref_ties(rc, llr_eq, d_max=d_max, use_pce=pce, use_vnr=vnr, threads=8)
        z[f"{mode}_drift"] = a["drift"]
        z[f"{mode}_bits"] = np.packbits(a["bits"], axis=1)
        z[f"{mode}_iterations"] = a["iterations"]
        z[f"{mode}_reasons"] = a["reasons"]
        z[f"{mode}_posteriors"] = a["posteriors"].astype(np.float32)
        z[f"{mode}_posteriors64_head"] = a["posteriors"][:, :64]
        z[f"{mode}_q_trace"] = a["q_trace"]
        z[f"{mode}_tie"] = tie
        print(name, mode, "iterations", a["iterations"].tolist(), "ties", int(tie.sum()))
    np.savez_compressed(os.path.join(HERE, name), **z)


def main():
    R = oracle.Reference()
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kats(R), f, indent=1)
    code = P.WORKLOADS["cfg1"].make_code()
    snr = P.snr_for_beta(0.95, code.rate())
    llr, x, _ = P.sample_frames(code, snr, P.FRAME_SEED, 0, 8)
    frames_reference(R, code, (llr * (1 - 2 * x.astype(np.float32))).astype(np.float32), 200,
                     "cfg1_reference.npz")
    lift = P.lift_protograph([[3, 3]], 1024, 1)
    snr = P.snr_for_beta(0.7, lift.rate())
    llr, _, _ = P.sample_frames(lift, snr, 77, 0, 8, all_zero=True)
    frames_reference(R, lift, llr, 200, "lift36_reference.npz")


if __name__ == "__main__":
    main()
