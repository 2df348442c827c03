"""Key-rate accounting (paper_2507_03509_b200/qkd.py) against the worked
examples and invariants of SPEC.md's qkd-metrics module;
the reference's qkd_metrics.cpp is not in the mounted tree."""
import math

import pytest

from paper_2507_03509_b200 import qkd

B2B = dict(transmittance_override=1.0, eta=1.0, nu_el=0.0, xi=0.0)


def test_mutual_information_examples():
    p = qkd.QkdSystemParams(v_a=3.0, mu=2, **B2B)
    assert qkd.mutual_information(p) == pytest.approx(math.log2(2.5), abs=1e-12)
    assert qkd.mutual_information(qkd.QkdSystemParams(v_a=1e-12, **B2B)) == pytest.approx(0.0, abs=1e-9)
    vals = [qkd.mutual_information(qkd.QkdSystemParams(v_a=v)) for v in (0.5, 1, 2, 4, 8)]
    assert all(a < b for a, b in zip(vals, vals[1:]))
    # homodyne is half the heterodyne log of the same ratio form
    ph = qkd.QkdSystemParams(v_a=3.0, mu=1, **B2B)
    assert qkd.mutual_information(ph) > 0


def test_solve_va_round_trip():
    p = qkd.QkdSystemParams(v_a=3.0, mu=2, **B2B)
    assert qkd.solve_va_for_iab(math.log2(2.5), p) == pytest.approx(3.0, abs=1e-12)
    for mu in (1, 2):
        for va in (0.3, 2.0, 7.5):
            q = qkd.QkdSystemParams(v_a=va, mu=mu)
            assert qkd.solve_va_for_iab(qkd.mutual_information(q), q) == pytest.approx(va, rel=1e-9)
    with pytest.raises(ValueError):
        qkd.solve_va_for_iab(0.0, p)


def test_g_and_holevo_invariants():
    assert qkd.g_entropy(1.0) == 0.0
    xs = [1.0, 1.5, 2.0, 5.0, 50.0]
    gs = [qkd.g_entropy(x) for x in xs]
    assert all(g >= 0 for g in gs) and all(a < b for a, b in zip(gs, gs[1:]))
    # identity channel leaks nothing, for any receiver
    for eta in (0.4, 0.8, 1.0):
        for nu in (0.0, 0.01, 0.1):
            for va in (0.5, 3.0, 10.0):
                for mu in (1, 2):
                    p = qkd.QkdSystemParams(transmittance_override=1.0, xi=0.0, eta=eta, nu_el=nu, v_a=va, mu=mu)
                    assert abs(qkd.holevo_bound(p)) < 1e-9


def test_paper_operating_point_sign():
    # R = 1/50, beta = 0.95: V_A from I_AB = R / beta; chi_BE > 0 and a positive key
    p = qkd.operating_point(1 / 50, 0.95)
    assert qkd.mutual_information(p) == pytest.approx(0.02 / 0.95, rel=1e-12)
    chi = qkd.holevo_bound(p)
    assert chi > 0
    assert 0.95 * qkd.mutual_information(p) - chi - qkd.finite_size_penalty(p) > 0


def test_finite_size_penalty():
    p = qkd.QkdSystemParams(n_privacy=1e8)
    assert qkd.finite_size_penalty(p) == pytest.approx(4.1e-3, rel=0.01)
    vals = [qkd.finite_size_penalty(qkd.QkdSystemParams(n_privacy=n)) for n in (1e4, 1e6, 1e8, 1e12)]
    assert all(a > b for a, b in zip(vals, vals[1:]))
    with pytest.raises(ValueError):
        qkd.finite_size_penalty(qkd.QkdSystemParams(n_privacy=100))


def test_equations_1_to_3_examples():
    assert qkd.eq1(0.95, 1.0, 0.1, 0.01, 0.001) == 0.0
    assert qkd.eq1(0.95, 0.0, 0.02 / 0.95, 0.01, 0.0041) == pytest.approx(0.0059, abs=1e-15)
    assert qkd.decoder_throughput(1e6, 500, 1 / 50, 0.0) == pytest.approx(40.0)
    assert qkd.decoder_throughput(1e6, 500, 1 / 50, 1.0) == 0.0
    assert qkd.decoder_throughput(1e6, 250, 1 / 50, 0.0) == pytest.approx(2 * 40.0)
    assert qkd.eq3(1e6, 250, 2, 0.5, 0.004) == pytest.approx(4.0)
    assert qkd.eq3(1e6, 250, 1, 0.5, 0.004) == pytest.approx(2 * qkd.eq3(1e6, 250, 2, 0.5, 0.004))
    assert qkd.eq3(1e6, 250, 2, 1.0, 0.004) == 0.0


def test_evaluate_consistency():
    for beta, fer, d in ((0.93, 0.1, 40.0), (0.97, 0.6, 120.0)):
        b = qkd.evaluate(1 / 50, beta, fer, 1e6, d)
        q = qkd.operating_point(1 / 50, beta)
        assert b.skr_dec * q.mu * d / 1e6 == pytest.approx(b.skr, rel=1e-12)
        assert b.k_throughput == pytest.approx(qkd.decoder_throughput(1e6, d, 1 / 50, fer))
        b2 = qkd.evaluate(1 / 50, beta, fer, 1e6, 2 * d)
        assert b2.skr_dec == pytest.approx(b.skr_dec / 2) and b2.k_throughput == pytest.approx(b.k_throughput / 2)


def test_optimize_beta():
    R = qkd.SweepRecord
    assert qkd.optimize_beta([R(0.95, 0.1, 1.0)]) == (0.95, 0.95)
    assert qkd.optimize_beta([R(0.93, 0.1, 3.0), R(0.95, 0.3, 1.0), R(0.97, 0.2, 2.0)]) == (0.95, 0.93)
    assert qkd.optimize_beta([R(0.96, 0.5, 0.0), R(0.94, 0.5, 0.0)]) == (0.94, 0.94)
    with pytest.raises(ValueError):
        qkd.optimize_beta([])
