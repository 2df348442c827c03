"""Exploration of two-edge-type (MET-style) low-rate code designs for a
waterfall (FER < 1) region: prototype construction in numpy, decoded on the
GPU with PCE, FER vs beta.  Output: JSON lines."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2507_03509_b200 as P


def met2(N, R, f1, d1, p1, k2, seed):
    rng = np.random.default_rng(seed)
    M = int(N * (1 - R) + 0.5)
    n1 = int(f1 * N + 0.5)
    Mc, nc = M - n1, N - n1
    cnt = np.floor(np.array(p1) * nc + 0.5).astype(int)
    cnt[-1] = nc - cnt[:-1].sum()
    deg1 = np.repeat(d1, cnt)
    rng.shuffle(deg1)
    s1 = np.repeat(np.arange(nc), deg1)
    c1 = np.arange(s1.size) % Mc
    rng.shuffle(c1)
    s2 = np.arange(n1 * k2) % nc
    c2 = Mc + np.arange(n1 * k2) // k2
    rng.shuffle(s2)
    lists = [set() for _ in range(M)]
    for v, c in zip(s1.tolist(), c1.tolist()):
        lists[c].add(v)
    for v, c in zip(s2.tolist(), c2.tolist()):
        lists[c].add(v)
    for j in range(n1):
        lists[Mc + j].add(nc + j)
    return P.ParityCheckMatrix.from_check_lists(N, [sorted(c) for c in lists])


designs = [
    # name, f1, d1 degrees, probs, k2
    ("A_f.85_k3", 0.85, [2, 3], [0.5, 0.5], 3),
    ("G_f.733_k3", 0.7333, [2, 3], [0.5, 0.5], 3),
    ("H_f.75_d2_k3", 0.75, [2], [1.0], 3),
    ("I_f.70_k2", 0.70, [2, 3], [0.5, 0.5], 2),
    ("J_f.80_k3_d2", 0.80, [2], [1.0], 3),
]
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
F = 64
betas = [0.6, 0.7, 0.75, 0.8, 0.85, 0.9]
for name, f1, d1, p1, k2 in designs:
    code = met2(N, 0.1, f1, d1, p1, k2, 7)
    dec = P.BatchDecoder(code, max_slots=64)
    vd = code.var_degrees()
    cd = code.check_degrees()
    for beta in betas:
        snr = P.snr_for_beta(beta, code.rate())
        llr, x, s = P.sample_frames(code, snr, 99, 0, F)
        out = {}
        for et, (pce, vnr) in (("pce", (True, False)), ("vnr", (True, True))):
            r = dec.decode_batch(llr, P.DecodeConfig(d_max=200, use_pce=pce, use_vnr=vnr, q_mode=P.decoder.Q_ABS),
                                 syndrome=s)
            ok = np.all(r.bits == x, axis=1)
            out[et] = {"fer": float(1 - ok.mean()), "d_bar": float(r.iterations.mean()),
                       "undetected": int(np.sum((r.reasons == 0) & ~ok))}
        print(json.dumps({"design": name, "N": N, "beta": beta, "rate": code.rate(), "max_vdeg": int(vd.max()),
                          "max_cdeg": int(cd.max()), **out}), flush=True)
