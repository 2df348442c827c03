import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_03509_b200 as P
from paper_2507_03509_b200.decoder import Q_ABS
w = P.WORKLOADS["cfg2"]; code = w.make_code(); F = 64
dec = P.BatchDecoder(code, max_slots=F)
N, M = code.n_vars, code.n_checks
d_llr = torch.empty((F, N), dtype=torch.float32, device="cuda")
d_syn = torch.empty((F, (M + 31) // 32), dtype=torch.int32, device="cuda")
dec.sample_frames_device(P.snr_for_beta(0.95, code.rate()), P.FRAME_SEED, 0, F, d_llr, d_syn)
out = {"iterations": torch.zeros(F, dtype=torch.int32, device="cuda"), "reasons": torch.zeros(F, dtype=torch.uint8, device="cuda"),
       "bits": torch.zeros((F, (N + 31) // 32), dtype=torch.int32, device="cuda")}
cfg = P.DecodeConfig(d_max=500, use_pce=True, use_vnr=True, q_mode=Q_ABS)
s = torch.cuda.Stream()
for label, kw in [("own-stream", {}), ("torch-stream", {"stream": s.cuda_stream}), ("own-stream", {}),
                  ("torch-stream", {"stream": s.cuda_stream})]:
    dec.decode_batch(d_llr, cfg, syndrome=d_syn, packed=True, out=out, **kw)
    torch.cuda.synchronize()
    l0 = dec.launch_count()
    t0 = time.perf_counter()
    for _ in range(3):
        dec.decode_batch(d_llr, cfg, syndrome=d_syn, packed=True, out=out, **kw)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(label, "ms/step %.2f" % (dt * 1e3), "launches/step", (dec.launch_count() - l0) / 3,
          "iters", int(out["iterations"].sum()), "max it", int(out["iterations"].max()), flush=True)
