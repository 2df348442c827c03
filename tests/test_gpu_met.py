"""Parity on the FER < 1 code family (workloads met_s / met: the two-edge-type
construction with a core code, generate_met_core) against the compiled
reference (oracle/_ref): converging frames exercise PCE stops, which the
BASELINE construction (FER = 1 everywhere) never does."""
import os

import numpy as np
import pytest

from _parity import compare, ref_ties

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 8
ET_MODES = {"none": (False, False), "pce": (True, False), "vnr": (True, True)}


def _refcode(ref, code):
    ptr, var = code.csr()
    return ref.code_from_csr(code.n_vars, code.n_checks, ptr, var)


@pytest.fixture(scope="module")
def met_s(P):
    return P.WORKLOADS["met_s"].make_code()


@pytest.mark.parametrize("beta", [0.7, 0.8, 0.9])
@pytest.mark.parametrize("mode", list(ET_MODES))
def test_met_small_vs_reference(P, ref, met_s, beta, mode):
    """N = 8192: all three ET modes; at beta 0.7 / 0.8 most frames converge
    (PCE stops with the right codeword), at 0.9 most fail."""
    F = 24
    snr = P.snr_for_beta(beta, met_s.rate())
    llr, x, s = P.sample_frames(met_s, snr, P.FRAME_SEED, 0, F)
    leq = (llr * (1 - 2 * x.astype(np.float32))).astype(np.float32)
    pce, vnr = ET_MODES[mode]
    rc = _refcode(ref, met_s)
    r, tie = ref_ties(rc, leq, d_max=200, use_pce=pce, use_vnr=vnr, threads=THREADS)
    g = P.BatchDecoder(met_s, max_slots=32).decode_batch(leq, P.DecodeConfig(d_max=200, use_pce=pce, use_vnr=vnr),
                                                         want_posteriors=True)
    summary = compare(g, r, tie, min_nontie_frac=0.5, label=f"met_s beta={beta} {mode}")
    conv = int(np.sum(g.reasons == 0))
    print(f"met_s beta={beta} {mode}: {summary}, syndrome stops {conv}/{F}")
    if mode != "none" and beta <= 0.8:
        assert conv >= F // 2  # the family decodes here (FER < 1)
    # the same frames in true syndrome mode (L, s = Hx) give bits xor x
    gs = P.BatchDecoder(met_s, max_slots=32).decode_batch(llr, P.DecodeConfig(d_max=200, use_pce=pce, use_vnr=vnr,
                                                                              q_mode=P.decoder.Q_ABS), syndrome=s)
    ga = P.BatchDecoder(met_s, max_slots=32).decode_batch(leq, P.DecodeConfig(d_max=200, use_pce=pce, use_vnr=vnr,
                                                                              q_mode=P.decoder.Q_ABS))
    assert np.array_equal(gs.iterations, ga.iterations) and np.array_equal(gs.reasons, ga.reasons)
    assert np.array_equal(gs.bits ^ x, ga.bits)


def test_met_full_size_vs_reference(P, ref):
    """N = 2^20 at beta 0.85 (top of the waterfall): PCE per frame
    (converging frames: syndrome stops on the right codeword), and VNR+PCE statistically (per-frame VNR at this size is
    decided by q gaps near float resolution, as for cfg5): the paired mean
    iteration difference within its CI and the same stop reasons."""
    code = P.WORKLOADS["met"].make_code()
    F = 8
    snr = P.snr_for_beta(0.85, code.rate())
    llr, x, s = P.sample_frames(code, snr, P.FRAME_SEED, 0, F)
    leq = (llr * (1 - 2 * x.astype(np.float32))).astype(np.float32)
    rc = _refcode(ref, code)
    # frames converging after ~80 iterations near the threshold amplify a
    # one-ulp input change in their posteriors (rule 3) while their outcome
    # stays put: compared exactly on bits / iterations / reason, posteriors
    # at the drift-widened bar (this is not a BASELINE configuration)
    r, tie = ref_ties(rc, leq, chaotic_is_tie=False, d_max=200, use_pce=True, use_vnr=False, threads=THREADS)
    dec = P.BatchDecoder(code, max_slots=32)
    g = dec.decode_batch(leq, P.DecodeConfig(d_max=200, use_pce=True, use_vnr=False), want_posteriors=True)
    summary = compare(g, r, tie, min_nontie_frac=0.5, strict=False, label="met full pce")
    print("met full pce: reference one-ulp posterior drift per frame", np.round(r["drift"], 2).tolist())
    ok = (g.reasons == 0) & np.all(g.bits == 0, axis=1)  # all-zero-equivalent form: the codeword is 0
    print(f"met N=2^20 beta=0.85 pce: {summary}, decoded {int(ok.sum())}/{F}, iterations {g.iterations.tolist()}")
    assert ok.sum() >= F // 2
    rv = rc.decode_batch(leq.astype(np.float64), d_max=200, use_pce=True, use_vnr=True, threads=THREADS,
                         want_posteriors=False, want_q_trace=False)
    gv = dec.decode_batch(leq, P.DecodeConfig(d_max=200, use_pce=True, use_vnr=True))
    d = gv.iterations.astype(np.float64) - rv["iterations"]
    se = d.std(ddof=1) / np.sqrt(F)
    print(f"met N=2^20 beta=0.85 vnr: D_bar gpu {gv.iterations.mean():.2f} ref {rv['iterations'].mean():.2f}, "
          f"paired {d.mean():+.3f} +- {se:.3f}, reasons gpu {gv.reasons.tolist()} ref {rv['reasons'].tolist()}")
    assert abs(d.mean()) <= 1.96 * se + 0.5
    assert np.mean(gv.reasons == rv["reasons"]) >= 0.75
