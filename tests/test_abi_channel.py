"""C ABI surface and channel/input generation (CPU only)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2507_03509_b200 as P
from paper_2507_03509_b200 import _lib
from conftest import ROOT


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "bpdec.h")).read()
    decl = r"^\s*(?:int|void|const char\s*\*)\s+(bpdec_[a-z_0-9]+)\s*\("
    return sorted(set(re.findall(decl, text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _declared_symbols()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    # and the Python binding covers every declared entry point
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(declared) <= bound, set(declared) - bound
    assert lib.bpdec_abi_version() == 1


def test_stop_reason_names_match_reference():
    """to_string(StopReason) (decoder.cpp:10-17)."""
    assert [str(r) for r in P.StopReason] == ["syndrome_satisfied", "vnr_drop", "max_iterations"]


def test_no_cpu_fallback_without_gpu():
    """Decoder creation must fail loudly when no sm_100 device is present."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    code = P.ParityCheckMatrix.from_check_lists(3, [[0, 1, 2]])
    with pytest.raises(P.BpdecCudaError):
        P.BatchDecoder(code)


def test_config_validation_before_device():
    """decode validates its config like decoder.cpp:63-64 (status 3)."""
    lib = _lib.load()
    cfg = _lib.Config(0, 1, 0, 0, 30.0)
    st = lib.bpdec_decode_batch(None, 1, None, None, C.byref(cfg), 0, None, None, None, None, None, None)
    assert st == 3  # null decoder -> validation


def test_snr_for_beta_kats(ref):
    assert P.snr_for_beta(1.0, 0.02) == 0.028113826656066543
    assert P.snr_for_beta(0.95, 0.1) == 0.15711023728271978
    assert P.snr_for_beta(0.98, 0.02) == 0.028695733476277407
    assert P.snr_for_beta(0.5, 0.25) == 1.0
    for b, r in ((0.92, 0.1), (0.99, 0.05), (0.3, 0.5)):
        assert P.snr_for_beta(b, r) == ref.snr_for_beta(b, r)
    with pytest.raises(P.ValidationError):
        P.snr_for_beta(0.0, 0.1)
    with pytest.raises(P.ValidationError):
        P.snr_for_beta(0.5, 1.0)
    # monotone decreasing in beta
    s = [P.snr_for_beta(b, 0.1) for b in np.linspace(0.5, 1.0, 11)]
    assert all(a > b for a, b in zip(s, s[1:]))


def test_all_zero_frames_equal_reference_sample_block(ref, cfg1_code):
    """At x = 0 the generator is sample_block (channel.cpp:44-61) rounded to
    float32: identical draws for (seed, trial)."""
    snr = P.snr_for_beta(0.95, cfg1_code.rate())
    llr, x, s = P.sample_frames(cfg1_code, snr, 1234, 7, 3, all_zero=True)
    assert not x.any() and not s.any()
    for b in range(3):
        r = ref.sample_block(snr, cfg1_code.n_vars, 1234, 7 + b)
        assert np.array_equal(llr[b], r.astype(np.float32))


def test_syndrome_mode_frames(orc, cfg1_code):
    """x ~ Bern(1/2) keyed by (seed, frame, i); llr = float((2/s2)((1-2x)+s g));
    s = Hx; the restatement in oracle.c agrees bit for bit."""
    snr = P.snr_for_beta(0.9, cfg1_code.rate())
    llr, x, s = P.sample_frames(cfg1_code, snr, 99, 100, 4)
    assert 0.45 < x.mean() < 0.55
    for b in range(4):
        ol, ox = orc.sample_frame(cfg1_code.n_vars, snr, 99, 100 + b)
        assert np.array_equal(ol, llr[b]) and np.array_equal(ox, x[b])
        assert np.array_equal(cfg1_code.syndrome(x[b]), s[b])
    # the noise is the reference's NoiseStream for (seed, frame): where x = 0
    # the syndrome-mode LLR equals the all-zero LLR bit for bit
    l0, _, _ = P.sample_frames(cfg1_code, snr, 99, 100, 1, all_zero=True)
    z = x[0] == 0
    assert np.array_equal(llr[0][z], l0[0][z])


def test_frames_moments(cfg1_code):
    """mean(llr) ~ 2 snr, var ~ 4 snr for the all-zero word."""
    snr = 0.5
    llr, _, _ = P.sample_frames(cfg1_code, snr, 3, 0, 64, all_zero=True)
    v = llr.astype(np.float64).ravel()
    se = np.sqrt(4 * snr / v.size)
    assert abs(v.mean() - 2 * snr) < 4 * se
    assert abs(v.var() - 4 * snr) < 0.02 * 4 * snr


def test_frames_are_sharding_invariant(cfg1_code):
    """Frame f depends only on (seed, f): generating [0, 8) equals [0,3)+[3,8)."""
    a = P.sample_frames(cfg1_code, 0.3, 5, 0, 8)
    b1 = P.sample_frames(cfg1_code, 0.3, 5, 0, 3)
    b2 = P.sample_frames(cfg1_code, 0.3, 5, 3, 5)
    for k in range(3):
        assert np.array_equal(a[k], np.concatenate([b1[k], b2[k]]))
