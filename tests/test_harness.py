"""Monte-Carlo harness (≙ run_trials, channel.cpp:74-156) and puncturing
(≙ apply_puncture, puncture.cpp:16-48)."""
import numpy as np
import pytest

import paper_2507_03509_b200 as P


@pytest.mark.parametrize("target,seed", [(0.6, 7), (0.55, 1), (0.75, 99)])
def test_apply_puncture_equals_reference(ref, lift36, target, seed):
    ptr, var = lift36.csr()
    rc = ref.code_from_csr(lift36.n_vars, lift36.n_checks, ptr, var)
    m = P.apply_puncture(lift36, target, seed)
    rp, eff = rc.apply_puncture(target, seed)
    assert np.array_equal(m.punctured, rp) and m.effective_rate == eff
    assert np.all(np.diff(m.punctured) > 0)
    assert np.all(lift36.var_degrees()[m.punctured] >= 2)  # degree-1 never punctured


def test_apply_puncture_spec_examples(cfg1_code):
    # SPEC.md: target = rate -> empty; N=1000, M=800, target 1/4 -> 200 positions
    assert P.apply_puncture(cfg1_code, cfg1_code.rate(), 3).empty()
    rng = np.random.default_rng(0)
    lists = [sorted(rng.choice(1000, size=4, replace=False).tolist()) for _ in range(800)]
    h = P.ParityCheckMatrix.from_check_lists(1000, lists)
    m = P.apply_puncture(h, 0.25, 5)
    assert m.punctured.size == 200 and m.effective_rate == pytest.approx(0.25)
    with pytest.raises(P.ValidationError, match="can only raise the rate"):
        P.apply_puncture(h, 0.1, 1)
    with pytest.raises(P.ValidationError):
        P.apply_puncture(h, 1.0, 1)


def test_wilson_interval_matches_reference_formula():
    for k, n in ((0, 10), (3, 10), (10, 10), (512, 1000), (1, 1)):
        lo, hi = P.wilson_interval(k, n)
        z = 1.959963984540054
        p = k / n
        d = 1 + z * z / n
        c = (p + z * z / (2 * n)) / d
        h = z * np.sqrt(p * (1 - p) / n + z * z / (4 * n * n)) / d
        assert lo == pytest.approx(max(0.0, c - h), abs=1e-15) and hi == pytest.approx(min(1.0, c + h), abs=1e-15)


@pytest.mark.gpu
def test_run_trials_block_invariance(lift36):
    """Prefix-exact stop rule: statistics do not depend on the device batch
    size (≙ worker-count invariance, channel.hpp:66-71, SPEC acceptance #8)."""
    dec = P.BatchDecoder(lift36, max_slots=256)
    cfg = P.DecodeConfig(d_max=200, use_pce=True, use_vnr=True)
    snr = P.snr_for_beta(0.7, lift36.rate())
    for stop in (P.StopRule(50, 10000), P.StopRule(0, 300)):
        a = P.run_trials(dec, snr, cfg, stop, 3, block=64)
        b = P.run_trials(dec, snr, cfg, stop, 3, block=256)
        c = P.run_trials(dec, snr, cfg, stop, 3, block=37)
        assert a == b == c
        if stop.min_frame_errors:
            assert a.frame_errors == 50 and not a.hit_max_frames
        else:
            assert a.frames == 300 and a.hit_max_frames


@pytest.mark.gpu
@pytest.mark.parametrize("beta,et", [(0.6, "pce"), (0.7, "pce"), (0.7, "vnr"), (0.8, "vnr")])
def test_run_trials_vs_reference(ref, lift36, beta, et):
    """GPU run_trials against the reference's own run_trials on the same
    seeds (the reference decodes double LLRs, the GPU their float32
    rounding): FER and mean iterations agree within the Wilson interval /
    a few percent, SPEC acceptance #5/#6 trends hold."""
    ptr, var = lift36.csr()
    rc = ref.code_from_csr(lift36.n_vars, lift36.n_checks, ptr, var)
    use_vnr = et == "vnr"
    r = rc.run_trials(beta, d_max=200, use_pce=True, use_vnr=use_vnr, min_frame_errors=0, max_frames=512, seed=11,
                      workers=8)
    dec = P.BatchDecoder(lift36, max_slots=256)
    g = P.run_trials(dec, P.snr_for_beta(beta, lift36.rate()), P.DecodeConfig(d_max=200, use_pce=True, use_vnr=use_vnr),
                     P.StopRule(0, 512), 11)
    assert g.frames == r["frames"] == 512
    assert abs(g.frame_errors - r["frame_errors"]) <= max(8, 0.04 * r["frame_errors"])
    assert g.fer_ci_low <= r["fer"] <= g.fer_ci_high
    assert abs(g.d_bar - r["d_bar"]) <= 0.06 * r["d_bar"] + 0.5
    assert g.stops_syndrome + g.stops_vnr + g.stops_max_iter == g.frames


@pytest.mark.gpu
def test_run_trials_punctured_and_trends(lift36):
    """Puncturing raises FER; FER is monotone non-increasing in D_max on the
    same seeds (SPEC acceptance #5); VNR lowers mean iterations (#6 trend)."""
    dec = P.BatchDecoder(lift36, max_slots=256)
    snr = P.snr_for_beta(0.65, lift36.rate())
    stop = P.StopRule(0, 512)
    fers = [P.run_trials(dec, snr, P.DecodeConfig(d_max=d), stop, 5).fer for d in (10, 50, 200)]
    assert fers[0] >= fers[1] >= fers[2]
    pce = P.run_trials(dec, snr, P.DecodeConfig(d_max=200), stop, 5)
    vnr = P.run_trials(dec, snr, P.DecodeConfig(d_max=200, use_vnr=True), stop, 5)
    assert vnr.d_bar < pce.d_bar
    mask = P.apply_puncture(lift36, 0.55, 9)
    punct = P.run_trials(dec, snr, P.DecodeConfig(d_max=200), stop, 5, mask=mask)
    assert punct.fer >= pce.fer
