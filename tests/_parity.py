"""Parity helpers: the tie rule of SURVEY §8(c) and the comparison bar of
BASELINE.json's north star (identical hard decisions / termination iteration /
reason on frames away from ties; posteriors within 1e-4 relative)."""
from __future__ import annotations

import numpy as np

POST_RTOL = 1e-4   # north star: "float32 LLR tolerance 1e-4 relative"
POST_ATOL = 1e-4   # LLR units, for posteriors near zero


def ulp_up(llr32: np.ndarray) -> np.ndarray:
    return np.nextafter(llr32.astype(np.float32), np.float32(np.inf)).astype(np.float32)


def ref_ties(refc, llr32, **kw):
    """Frames whose reference outcome changes when every float32 LLR moves by
    one ulp (the reference's own sensitivity; SURVEY §8c tie rule)."""
    a = refc.decode_batch(llr32.astype(np.float64), want_posteriors=True, **kw)
    b = refc.decode_batch(ulp_up(llr32).astype(np.float64), want_posteriors=False, **kw)
    tie = ((a["bits"] != b["bits"]).any(axis=1) | (a["iterations"] != b["iterations"]) |
           (a["reasons"] != b["reasons"]))
    return a, tie


def compare(gpu, ref, tie, *, post=True, min_nontie_frac=0.5, label=""):
    """Asserts the parity bar on non-tie frames; returns a summary dict."""
    B = len(ref["iterations"])
    bad = []
    for f in range(B):
        if tie[f]:
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
            g = gpu.posteriors[f].astype(np.float64)
            r = ref["posteriors"][f]
            if not np.allclose(g, r, rtol=POST_RTOL, atol=POST_ATOL):
                err = np.max(np.abs(g - r) / (np.abs(r) * POST_RTOL + POST_ATOL))
                bad.append((f, "posteriors", float(err)))
    nontie = int(B - tie.sum())
    assert not bad, f"{label}: parity failures on non-tie frames: {bad[:8]}"
    assert nontie >= min_nontie_frac * B, f"{label}: too many tie frames ({int(tie.sum())}/{B})"
    return {"frames": B, "ties": int(tie.sum()), "checked": nontie}
