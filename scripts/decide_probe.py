#!/usr/bin/env python3
"""k_decide cost by ET mode (ncu target): cfg2 code, 64 device-generated frames, D_max 6."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_03509_b200 as P  # noqa: E402
from paper_2507_03509_b200.decoder import Q_ABS  # noqa: E402
w = P.WORKLOADS["cfg2"]; code = w.make_code(); frames = 64
dec = P.BatchDecoder(code, max_slots=frames)
N, M = code.n_vars, code.n_checks
d_llr = torch.empty((frames, N), dtype=torch.float32, device="cuda")
d_syn = torch.empty((frames, (M + 31) // 32), dtype=torch.int32, device="cuda")
dec.sample_frames_device(P.snr_for_beta(0.95, code.rate()), P.FRAME_SEED, 0, frames, d_llr, d_syn)
out = {"iterations": torch.zeros(frames, dtype=torch.int32, device="cuda"),
       "reasons": torch.zeros(frames, dtype=torch.uint8, device="cuda"),
       "bits": torch.zeros((frames, (N + 31) // 32), dtype=torch.int32, device="cuda")}
for pce, vnr in ((True, False), (False, True), (False, False)):
    cfg = P.DecodeConfig(d_max=6, use_pce=pce, use_vnr=vnr, q_mode=Q_ABS)
    dec.decode_batch(d_llr, cfg, syndrome=d_syn, packed=True, out=out)
torch.cuda.synchronize()
