#!/usr/bin/env python3
"""Short, deterministic decode used as the ncu capture target: config-2 code,
64 device-generated frames, PCE-ET, D_max=6 (every frame runs 6 iterations).
Third argument "vnr": the bench decode instead (VNR+PCE, the workload's D_max);
"stream": VNR+PCE with the frames streaming through a quarter of the slots."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_03509_b200 as P  # noqa: E402
from paper_2507_03509_b200.decoder import Q_ABS  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 64
w = P.WORKLOADS[wl]
code = w.make_code()
dec = P.BatchDecoder(code, max_slots=frames)
N, M = code.n_vars, code.n_checks
d_llr = torch.empty((frames, N), dtype=torch.float32, device="cuda")
d_syn = torch.empty((frames, (M + 31) // 32), dtype=torch.int32, device="cuda")
dec.sample_frames_device(P.snr_for_beta(0.95, code.rate()), P.FRAME_SEED, 0, frames, d_llr, d_syn)
out = {"iterations": torch.zeros(frames, dtype=torch.int32, device="cuda"),
       "reasons": torch.zeros(frames, dtype=torch.uint8, device="cuda"),
       "bits": torch.zeros((frames, (N + 31) // 32), dtype=torch.int32, device="cuda")}
mode = sys.argv[3] if len(sys.argv) > 3 else "pce6"
if mode == "stream":  # frames stream through a quarter of the slots
    dec = P.BatchDecoder(code, max_slots=max(32, frames // 4))
cfg = (P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=True, q_mode=Q_ABS) if mode in ("vnr", "stream")
       else P.DecodeConfig(d_max=6, use_pce=True, use_vnr=False, q_mode=Q_ABS))
r = dec.decode_batch(d_llr, cfg, syndrome=d_syn,
                     packed=True, out=out)
torch.cuda.synchronize()
print("iterations", int(out["iterations"].sum().item()), "launches", dec.launch_count())
