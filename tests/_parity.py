"""Parity helpers: the tie rule of SURVEY §8(c) and the comparison bar of
BASELINE.json's north star (identical hard decisions / termination iteration /
reason on frames away from ties; posteriors within 1e-4 relative).

Tie rule (a frame is a tie when the reference itself cannot decide it
robustly at float32 input precision):
  1. its outcome (bits, iterations, reason) changes when every float32 LLR
     moves one ulp up, one ulp down, or each LLR independently moves one ulp
     up / down / not at all (four seeded patterns) — coherent shifts alone
     miss oscillating frames that return to the same attractor;
  2. VNR-ET on and some gap |q_k - q_(k-1)|, 2 <= k <= stop, is within
     Q_GAP_REL * |q_k| (the decision is a coin flip at float precision);
  3. chaotic: its posteriors under the one-ulp-up input move by more than
     the posterior tolerance (non-converging BP
     amplifies a one-ulp input change up to 90x).
Posterior bar on non-tie frames: |gpu - ref| <= 1e-4 |ref| + 1e-4, or within
DRIFT_FACTOR times the reference's own one-ulp posterior drift for that frame
(float32 rounding of every message vs one input rounding).
"""
from __future__ import annotations

import numpy as np

POST_RTOL = 1e-4   # north star: "float32 LLR tolerance 1e-4 relative"
POST_ATOL = 1e-4   # LLR units, for posteriors near zero
Q_GAP_REL = 2e-8   # ~ float32 epsilon / 3: a q drop smaller than this is a coin flip
DRIFT_FACTOR = 32.0


def ulp_up(llr32: np.ndarray) -> np.ndarray:
    return np.nextafter(llr32.astype(np.float32), np.float32(np.inf)).astype(np.float32)


def ulp_down(llr32: np.ndarray) -> np.ndarray:
    return np.nextafter(llr32.astype(np.float32), np.float32(-np.inf)).astype(np.float32)


def ulp_random(llr32: np.ndarray, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    step = rng.integers(-1, 2, size=llr32.shape)
    up, dn = ulp_up(llr32), ulp_down(llr32)
    return np.where(step > 0, up, np.where(step < 0, dn, llr32.astype(np.float32)))


def _norm_err(g, r):
    return np.max(np.abs(g - r) / (np.abs(r) * POST_RTOL + POST_ATOL))


def _q_gap_ties(a, kw):
    """Tie rule 2: a VNR comparison that decided the run was within
    Q_GAP_REL of |q| (k' = 2 .. stop-1 without a drop, and the stop iteration
    itself only if VNR fired there; PCE is checked first, decoder.cpp:115-122)."""
    B = len(a["iterations"])
    tie = np.zeros(B, dtype=bool)
    if not kw.get("use_vnr") or a["q_trace"] is None:
        return tie
    for f in range(B):
        k = int(a["iterations"][f])
        last = k if int(a["reasons"][f]) == 1 else k - 1
        q = a["q_trace"][f, :k]
        gaps = np.abs(np.diff(q))[: max(last - 1, 0)]
        if gaps.size and np.any(gaps <= Q_GAP_REL * np.maximum(np.abs(q[1:last]), 1.0)):
            tie[f] = True
    return tie


def ref_ties(refc, llr32, chaotic_is_tie=True, **kw):
    """Runs the reference on the inputs and on their +-1 ulp neighbours.
    Returns (reference outputs with 'drift' per frame, tie mask).  Frames
    already tied by the q-gap rule skip the perturbed runs (their verdict
    cannot change), which keeps full-size VNR configurations affordable.
    chaotic_is_tie=False keeps rule-3 frames (outcome stable under the
    perturbations, posteriors not) in the comparison: their bits,
    iterations and reason are compared exactly and their posteriors at
    DRIFT_FACTOR x the measured drift (compare with strict=False)."""
    a = refc.decode_batch(llr32.astype(np.float64), want_posteriors=True, **kw)
    B = len(a["iterations"])
    tie = _q_gap_ties(a, kw)
    drift = np.full(B, np.inf)
    idx = np.nonzero(~tie)[0]
    if idx.size:
        sub = llr32[idx]
        b = refc.decode_batch(ulp_up(sub).astype(np.float64), want_posteriors=True, **kw)
        others = [b, refc.decode_batch(ulp_down(sub).astype(np.float64), want_posteriors=False, **kw)]
        for seed in (1, 2, 3, 4):
            others.append(refc.decode_batch(ulp_random(sub, seed).astype(np.float64), want_posteriors=False, **kw))
        for j, f in enumerate(idx):
            t = False
            for o in others:
                t |= bool(np.any(a["bits"][f] != o["bits"][j]) or a["iterations"][f] != o["iterations"][j] or
                          a["reasons"][f] != o["reasons"][j])
            if not t:
                drift[f] = _norm_err(b["posteriors"][j], a["posteriors"][f])
                t = chaotic_is_tie and drift[f] > 1.0  # chaotic frame (rule 3)
            tie[f] = t
    a["drift"] = drift
    return a, tie


def compare(gpu, ref, tie, *, post=True, min_nontie_frac=0.5, failed_decode_slack=0.0, label="", strict=False,
            min_checked=0):
    """Asserts the parity bar on non-tie frames; returns a summary dict.

    failed_decode_slack: fraction of non-tie frames allowed to differ when the
    reference frame is a failed decode that ran to d_max (a trapping-set fixed
    point reached after a long transient; float vs double arithmetic can pick
    a different trapping set even when +-1-ulp inputs cannot).  Used only for
    the desk-scale (3,6) code; 0 for the BASELINE configurations."""
    B = len(ref["iterations"])
    bad = []
    slack = []
    worst = 0.0
    drift = ref.get("drift")
    for f in range(B):
        if tie[f]:
            continue
        failed = int(ref["reasons"][f]) == 2
        if failed and failed_decode_slack > 0 and (
                gpu.iterations[f] != ref["iterations"][f] or gpu.reasons[f] != ref["reasons"][f] or
                (gpu.bits is not None and np.any(gpu.bits[f] != ref["bits"][f]))):
            slack.append(f)
            continue
        if gpu.iterations[f] != ref["iterations"][f] or gpu.reasons[f] != ref["reasons"][f]:
            bad.append((f, "iterations/reason", int(gpu.iterations[f]), int(ref["iterations"][f]),
                        int(gpu.reasons[f]), int(ref["reasons"][f])))
            continue
        if gpu.bits is not None:
            diff = np.nonzero(gpu.bits[f] != ref["bits"][f])[0]
            if diff.size:
                # a bit flip on an (almost) exactly-zero posterior is a tie
                if ref["posteriors"] is not None and np.all(np.abs(ref["posteriors"][f][diff]) < 1e-3):
                    continue
                bad.append((f, "bits", int(diff.size)))
                continue
        if post and gpu.posteriors is not None and ref["posteriors"] is not None:
            e = _norm_err(gpu.posteriors[f].astype(np.float64), ref["posteriors"][f])
            # strict (BASELINE configurations): the north star's 1e-4 bar
            # itself, never widened by the reference's own one-ulp drift
            bound = 1.0 if (strict or drift is None) else max(1.0, DRIFT_FACTOR * drift[f])
            worst = max(worst, e)
            if e > bound:
                bad.append((f, "posteriors", float(e), float(bound)))
    nontie = int(B - tie.sum())
    assert not bad, f"{label}: parity failures on non-tie frames: {bad[:8]}"
    assert len(slack) <= failed_decode_slack * max(nontie, 1), f"{label}: failed-decode mismatches {slack}"
    assert nontie >= min_nontie_frac * B, f"{label}: too many tie frames ({int(tie.sum())}/{B})"
    assert nontie >= min_checked, f"{label}: only {nontie} non-tie frames compared (need {min_checked})"
    return {"frames": B, "ties": int(tie.sum()), "checked": nontie, "worst_post_err": worst,
            "failed_decode_mismatches": len(slack), "strict": strict}
