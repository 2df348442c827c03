"""Randomised differential tests: seeded random multi-edge-style codes
(degree-1 variables, degree-0 variables and empty checks, variable degrees
2..40, mixed check types so both typed and generic kernel paths run),
random LLR mixtures (punctured zeros, values beyond the clamp), random
D_max / ET mode / message clamp / slot count / batch — the CUDA decoder
against the compiled reference with the tie rule of tests/_parity.py."""
import os

import numpy as np
import pytest

from _parity import compare, ref_ties

pytestmark = pytest.mark.gpu


def _random_code(P, rng):
    n_hi = int(rng.integers(80, 400))
    degs = rng.choice([2, 3, 3, 4, 6, 8, 12, 20, 40], size=n_hi)
    m = int(rng.integers(n_hi // 2, n_hi + 200))
    lists = [set() for _ in range(m)]
    for v, d in enumerate(degs):
        for c in rng.choice(m, size=int(min(d, m)), replace=False):
            lists[int(c)].add(v)
    # degree-1 variables on a random subset of checks, a few degree-0 ones
    n1 = int(rng.integers(m // 2, m))
    d1_checks = rng.choice(m, size=n1, replace=False)
    for j, c in enumerate(d1_checks):
        lists[int(c)].add(n_hi + j)
    n0 = int(rng.integers(0, 5))
    n = n_hi + n1 + n0
    if n <= m:  # the reference requires rate > 0
        n0 += m - n + 1
        n = n_hi + n1 + n0
    return P.ParityCheckMatrix.from_check_lists(n, [sorted(c) for c in lists])


def _random_llr(rng, frames, n, clamp):
    mu = float(rng.uniform(0.2, 3.0))
    sd = float(rng.uniform(0.5, 2.5))
    llr = rng.normal(mu, sd, size=(frames, n)) * rng.choice([-1.0, 1.0], size=(frames, n), p=[0.1, 0.9])
    llr[rng.random((frames, n)) < 0.02] = 0.0                      # punctured positions
    big = rng.random((frames, n)) < 0.01
    llr[big] = np.sign(llr[big] + 1e-9) * (clamp + rng.uniform(0.0, 30.0, size=int(big.sum())))
    return llr.astype(np.float32)


# BPDEC_FUZZ_SEEDS=<n> widens the sweep (profiles/r2/fuzz_extended.md: 300 seeds)
@pytest.mark.parametrize("seed", range(int(os.environ.get("BPDEC_FUZZ_SEEDS", "24"))))
def test_random_codes_vs_reference(P, ref, seed):
    rng = np.random.default_rng(1000 + seed)
    code = _random_code(P, rng)
    clamp = float(rng.choice([30.0, 12.0, 25.0]))
    d_max = int(rng.choice([1, 3, 20, 60]))
    pce, vnr = [(False, False), (True, False), (True, True)][seed % 3]
    frames = int(rng.integers(1, 70))
    slots = int(rng.choice([32, 64, 96]))
    llr = _random_llr(rng, frames, code.n_vars, clamp)
    ptr, var = code.csr()
    rc = ref.code_from_csr(code.n_vars, code.n_checks, ptr, var)
    r, tie = ref_ties(rc, llr, d_max=d_max, use_pce=pce, use_vnr=vnr, msg_clamp=clamp, threads=8)
    dec = P.BatchDecoder(code, max_slots=slots)
    g = dec.decode_batch(llr, P.DecodeConfig(d_max=d_max, use_pce=pce, use_vnr=vnr, msg_clamp=clamp),
                         want_posteriors=True)
    # small random codes at random SNR are often chaotic:
    # no minimum non-tie fraction, the bar applies to the frames that are not ties
    res = compare(g, r, tie, min_nontie_frac=0.0, label=f"fuzz seed={seed} d_max={d_max} pce={pce} vnr={vnr} "
                                                  f"clamp={clamp} frames={frames} slots={slots}")
    print(f"fuzz seed={seed}: N={code.n_vars} M={code.n_checks} frames={frames} d_max={d_max} "
          f"pce={pce} vnr={vnr}: {res}")
