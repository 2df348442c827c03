#!/usr/bin/env python3
"""ncu capture target: the lifted rate-0.1 protograph of scripts/qc_probe.py,
64 syndrome-mode frames, PCE with D_max = 6."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import paper_2507_03509_b200 as P  # noqa: E402
from paper_2507_03509_b200.decoder import Q_ABS  # noqa: E402
import qc_probe  # noqa: E402

code = P.lift_protograph(qc_probe.protograph(np.random.default_rng(7)), 10486, 11)
frames = 64
N, M = code.n_vars, code.n_checks
dec = P.BatchDecoder(code, max_slots=frames)
llr = torch.empty((frames, N), dtype=torch.float32, device="cuda")
syn = torch.empty((frames, (M + 31) // 32), dtype=torch.int32, device="cuda")
dec.sample_frames_device(P.snr_for_beta(0.95, code.rate()), P.FRAME_SEED, 0, frames, llr, syn)
r = dec.decode_batch(llr, P.DecodeConfig(d_max=6, use_pce=True, use_vnr=False, q_mode=Q_ABS), syndrome=syn,
                     packed=True)
torch.cuda.synchronize()
print("iterations", int(r.iterations.sum()))
