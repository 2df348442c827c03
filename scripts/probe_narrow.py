import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2507_03509_b200 as P
code = P.WORKLOADS["cfg1"].make_code()
llr, x, s, snr = P.sample_frames_beta(code, 0.2, 1.0, 808, 0, 96)
print("snr range", snr.min(), snr.max())
for pce, vnr in ((True, True), (True, False)):
    cfg = P.DecodeConfig(d_max=150, use_pce=pce, use_vnr=vnr, q_mode=P.decoder.Q_ABS)
    for nn in ("0", "1"):
        os.environ["BPDEC_NO_NARROW"] = nn
        for slots in (96, 32):
            r = P.BatchDecoder(code, max_slots=slots).decode_batch(llr, cfg, syndrome=s)
            print(pce, vnr, "no_narrow", nn, "slots", slots, np.bincount(r.iterations)[:40].nonzero()[0][:20], r.iterations[:24])
llr2, x2, s2 = P.sample_frames(code, P.snr_for_beta(0.95, code.rate()), 808, 0, 96)
cfg = P.DecodeConfig(d_max=150, use_pce=True, use_vnr=True, q_mode=P.decoder.Q_ABS)
for nn in ("0", "1"):
    os.environ["BPDEC_NO_NARROW"] = nn
    r = P.BatchDecoder(code, max_slots=96).decode_batch(llr2, cfg, syndrome=s2)
    print("fixed beta .95 no_narrow", nn, r.iterations[:32])
