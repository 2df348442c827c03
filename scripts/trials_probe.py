#!/usr/bin/env python3
"""Throughput of the GPU Monte-Carlo harness (bpdec_run_trials ≙ run_trials, channel.cpp:74-156) against the
stream decode of the same code: edge-updates/s including on-device frame generation.
usage: python scripts/trials_probe.py [workload] [beta] [max_frames]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_03509_b200 as P  # noqa: E402
from paper_2507_03509_b200.decoder import Q_RAW  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "met"
    beta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.87
    frames = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
    w = P.WORKLOADS[wl]
    code = w.make_code()
    dec = P.BatchDecoder(code, max_slots=384)
    snr = P.snr_for_beta(beta, code.rate())
    out = {}
    for name, vnr in (("pce", False), ("vnr", True)):
        cfg = P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=vnr, q_mode=Q_RAW)
        stop = P.StopRule(min_frame_errors=10 ** 9, max_frames=frames)
        P.run_trials(dec, snr, cfg, P.StopRule(min_frame_errors=10 ** 9, max_frames=128), 7, block=64)  # warm
        t0 = time.perf_counter()
        st = P.run_trials(dec, snr, cfg, stop, 7, block=int(os.environ.get("BLOCK", "0")) or None)
        dt = time.perf_counter() - t0
        out[name] = {"frames": st.frames, "fer": st.fer, "d_bar": st.d_bar, "seconds": dt,
                     "edge_updates_per_s": st.iteration_sum * code.n_edges / dt}
    print(json.dumps({"workload": w.name, "beta": beta, **out}))


if __name__ == "__main__":
    main()
