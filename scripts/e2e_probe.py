#!/usr/bin/env python3
"""Where the e2e time goes (cfg2, 64 frames, VNR+PCE): wall time per decode
call with device or pinned-host inputs (staged one call ahead) and outputs."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_03509_b200 as P  # noqa: E402
from paper_2507_03509_b200.decoder import Q_ABS  # noqa: E402

w = P.WORKLOADS["cfg2"]; code = w.make_code(); F = 64
N, M = code.n_vars, code.n_checks; MW, NW = (M + 31) // 32, (N + 31) // 32
dec = P.BatchDecoder(code, max_slots=F)
d_llr = torch.empty((F, N), dtype=torch.float32, device="cuda")
d_syn = torch.empty((F, MW), dtype=torch.int32, device="cuda")
dec.sample_frames_device(P.snr_for_beta(0.95, code.rate()), P.FRAME_SEED, 0, F, d_llr, d_syn)
h_llr = [torch.empty((F, N), dtype=torch.float32, pin_memory=True) for _ in range(2)]
h_syn = [torch.empty((F, MW), dtype=torch.int32, pin_memory=True) for _ in range(2)]
for i in range(2):
    h_llr[i].copy_(d_llr); h_syn[i].copy_(d_syn)
cfg = P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=True, q_mode=Q_ABS)
outs = {"dev": {"iterations": torch.zeros(F, dtype=torch.int32, device="cuda"),
                "reasons": torch.zeros(F, dtype=torch.uint8, device="cuda"),
                "bits": torch.zeros((F, NW), dtype=torch.int32, device="cuda")},
        "host": {"iterations": torch.zeros(F, dtype=torch.int32, pin_memory=True),
                 "reasons": torch.zeros(F, dtype=torch.uint8, pin_memory=True),
                 "bits": torch.zeros((F, NW), dtype=torch.int32, pin_memory=True)}}
K = 15
for inp in ("dev", "host"):
    for outk in ("dev", "host"):
        out = outs[outk]
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if inp == "host":
                dec.stage_inputs(h_llr[0], h_syn[0])
            for k in range(K):
                if inp == "host":
                    if k + 1 < K:
                        dec.stage_inputs(h_llr[(k + 1) % 2], h_syn[(k + 1) % 2])
                    dec.decode_batch(h_llr[k % 2], cfg, syndrome=h_syn[k % 2], packed=True, out=out)
                else:
                    dec.decode_batch(d_llr, cfg, syndrome=d_syn, packed=True, out=out)
                int(out["iterations"].sum().item())
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / K * 1e3
        print(f"in={inp:4s} out={outk:4s} {dt:.3f} ms/call")

# device inputs with an unrelated 276 MB H2D copy in flight during each call
# (is the staged-input cost the DMA's interference with the decode?)
junk_h = torch.empty((F, N), dtype=torch.float32, pin_memory=True)
junk_d = torch.empty((F, N), dtype=torch.float32, device="cuda")
cs = torch.cuda.Stream()
out = outs["dev"]
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        with torch.cuda.stream(cs):
            junk_d.copy_(junk_h, non_blocking=True)
        dec.decode_batch(d_llr, cfg, syndrome=d_syn, packed=True, out=out)
        int(out["iterations"].sum().item())
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / K * 1e3
print(f"in=dev  out=dev  + concurrent 276 MB H2D: {dt:.3f} ms/call")
