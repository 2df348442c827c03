"""Accuracy of the phi-domain magnitude map used by the check kernel
(csrc/phi.cuh), emulated on the CPU in float32 with correctly rounded exp2 /
log2 standing in for MUFU.EX2 / MUFU.LG2 (whose ~2-ulp error comes on top).
Also re-derives the polynomial fits the header quotes."""
import re

import numpy as np
import pytest

from conftest import ROOT


def _coeffs():
    src = open(f"{ROOT}/paper_2507_03509_b200/csrc/phi.cuh").read()
    body = src[src.index("float phi(float x)"):]
    nums = [float(x) for x in re.findall(r"(-?\d+\.\d+(?:e-?\d+)?)f", body)]
    # order in the source: log2e, a4..a1 (doubled), b4..b1, ln2 ..., 1.0 split
    return nums


def phi_emulated(x):
    """float32 re-statement of dev::phi with exact exp2/log2."""
    f = np.float32
    x = np.asarray(x, dtype=np.float32)
    with np.errstate(all="ignore"):
        t = np.exp2(x * f(-1.4426950408889634)).astype(np.float32)
        w = (t * t).astype(np.float32)
        a = f(2.0 * 0.14783698262526393)
        a = (a * w + f(2.0 * 0.1383879360711249)).astype(np.float32)
        a = (a * w + f(2.0 * 0.2002081579507349)).astype(np.float32)
        a = (a * w + f(2.0 * 0.3333303414682521)).astype(np.float32)
        hi = (t * (a * w + f(2.0))).astype(np.float32)
        z = (x * x).astype(np.float32)
        b = f(-2.1672081029454006e-05)
        b = (b * z + f(0.0003380189508581495)).astype(np.float32)
        b = (b * z + f(-0.0048599077080608115)).astype(np.float32)
        b = (b * z + f(0.08333320963387135)).astype(np.float32)
        lo = (np.log2(x).astype(np.float32) * f(-0.6931471805599453) + (b * z + f(0.6931471805599453))).astype(
            np.float32)
    return np.where(x < 1, lo, hi)


def phi_exact(x):
    x = np.asarray(x, dtype=np.float64)
    with np.errstate(all="ignore"):
        return np.log1p(2.0 / np.expm1(x))


def test_phi_relative_accuracy():
    x = np.concatenate([np.geomspace(1e-6, 1.0, 20001), np.linspace(1.0, 40.0, 40001)]).astype(np.float32)
    got = phi_emulated(x).astype(np.float64)
    ref = phi_exact(x.astype(np.float64))
    rel = np.abs(got - ref) / ref
    # Polynomial + float32 rounding: <= 6e-7 for x <= 10.  For large x the
    # rounding of x*log2(e) perturbs the exponent like a relative change of x
    # by ~6e-8, the same as x's own float32 rounding (phi's condition number
    # is ~x there): bound 6e-7 + 6e-8*x.  MUFU adds ~2 ulp on the hardware.
    assert (rel <= 6e-7 + 6e-8 * x).all(), rel.max()
    assert rel[x <= 10].max() < 6e-7


def test_phi_involution_and_limits():
    x = np.linspace(0.05, 25.0, 5000).astype(np.float32)
    back = phi_emulated(phi_emulated(x)).astype(np.float64)
    # phi(phi(x)) = x; error grows like x * eps for large x (exp2 argument rounding)
    assert np.max(np.abs(back - x) / np.maximum(x, 1.0)) < 2e-6
    with np.errstate(all="ignore"):
        assert phi_emulated(np.float32(0.0)) == np.inf
        assert phi_emulated(np.float32(np.inf)) == 0.0


def test_saturated_check_outputs():
    """Two inputs at the +-30 clamp: exact 29.306852819440055 (float tanh
    domain would give inf -> 30, the reference's double gives 29.306686)."""
    p30 = phi_emulated(np.float32(30.0))
    out = phi_emulated(np.float32(p30 + p30))
    assert out == pytest.approx(29.306852819440055, rel=2e-7)


@pytest.mark.parametrize("a_split", [1.0])
def test_fit_errors_reproduce(a_split):
    """Least-squares fits on Chebyshev nodes: g(z) = -ln(tanh(x/2)/(x/2)) ~
    z*B3(z) on x < 1 and atanh(t)/t - 1 ~ w*A3(w) on x >= 1 (header values)."""
    zs = np.cos(np.linspace(0, np.pi, 800)) * 0.5 * a_split ** 2 + 0.5 * a_split ** 2
    zs = zs[zs > 1e-12]
    xs = np.sqrt(zs)
    g = -np.log(np.tanh(xs / 2) / (xs / 2))
    V = np.vstack([zs ** (k + 1) for k in range(4)]).T
    c, *_ = np.linalg.lstsq(V, g, rcond=None)
    assert np.max(np.abs(V @ c - g)) < 5e-9
    wmax = np.exp(-2 * a_split)
    ws = np.cos(np.linspace(0, np.pi, 800)) * 0.5 * wmax + 0.5 * wmax
    ws = ws[ws > 1e-14]
    h = np.arctanh(np.sqrt(ws)) / np.sqrt(ws) - 1
    V = np.vstack([ws ** (k + 1) for k in range(4)]).T
    c, *_ = np.linalg.lstsq(V, h, rcond=None)
    assert np.max(np.abs(V @ c - h)) < 2e-8


# ---- t domain (the shipped form; csrc/phi.cuh second half) -----------------
def _f(x):
    return np.asarray(x, dtype=np.float32)


def t_emulated_outputs(m, clamp=np.float32(30.0)):
    """float32 restatement of t_outputs<3, 3> (tdom, tf_pair, tmag) for
    degree-3 checks: m[..., 3] magnitudes -> out[..., 3], exact exp2 / log2
    standing in for MUFU.EX2 / MUFU.LG2."""
    f = np.float32
    with np.errstate(all="ignore"):
        t = np.exp2(_f(m) * f(-1.4426950408889634)).astype(np.float32)
        out = []
        for a, b in ((1, 2), (0, 2), (0, 1)):
            n = (t[..., a] + t[..., b]).astype(np.float32)
            d = (t[..., a].astype(np.float64) * t[..., b].astype(np.float64) + 1.0).astype(np.float32)  # fma
            mag = np.abs(((np.log2(d).astype(np.float32) - np.log2(n).astype(np.float32)).astype(np.float32)
                          * f(0.6931471805599453)).astype(np.float32))
            out.append(np.minimum(mag, clamp))
    return np.stack(out, axis=-1)


def exact_outputs(m, clamp=30.0):
    m = np.asarray(m, dtype=np.float64)
    th = np.tanh(m / 2)
    out = []
    for a, b in ((1, 2), (0, 2), (0, 1)):
        # 2 atanh(x y) through log1p of the complementary product (exact near saturation)
        ta, tb = np.exp(-m[..., a]), np.exp(-m[..., b])
        T = (ta + tb) / (1 + ta * tb)
        with np.errstate(divide="ignore"):
            out.append(np.minimum(-np.log(T), clamp))
    del th
    return np.stack(out, axis=-1)


def test_t_domain_accuracy_grid():
    """The t-domain check update stays within 2e-6 (abs + rel) of the exact
    value over magnitudes 0..30, including the saturation corner where the
    float tanh form collapses."""
    rng = np.random.default_rng(7)
    m = np.concatenate([
        rng.uniform(0, 30, size=(200000, 3)),
        rng.uniform(0, 1e-3, size=(20000, 3)),
        rng.uniform(25, 30, size=(20000, 3)),
        np.array([[30, 30, 30], [0, 5, 7], [0, 0, 0], [30, 1e-6, 12], [20, 20, 20]], dtype=np.float64),
    ]).astype(np.float32)
    got = t_emulated_outputs(m).astype(np.float64)
    want = exact_outputs(m.astype(np.float64))
    err = np.abs(got - want) / (1.0 + np.abs(want))
    assert err.max() < 2e-6, err.max()
    # a zero input makes the other outputs exactly zero (tanh 0 = 0 in the reference)
    z = t_emulated_outputs(_f([[0.0, 5.0, 7.0]]))
    assert z[0, 1] == 0.0 and z[0, 2] == 0.0 and abs(z[0, 0] - exact_outputs([[0.0, 5.0, 7.0]])[0, 0]) < 1e-5


def test_t_domain_beats_double_tanh_at_saturation():
    """At (30, 30) the reference's double tanh/atanh form is 5.7e-6 off the
    exact value; the float t domain is within 1e-6."""
    m = _f([[30.0, 30.0, 30.0]])
    got = float(t_emulated_outputs(m, clamp=np.float32(100.0))[0, 0])
    exact = float(exact_outputs(m.astype(np.float64), clamp=100.0)[0, 0])
    ref = float(2 * np.arctanh(np.tanh(15.0) * np.tanh(15.0)))
    assert abs(got - exact) < 1e-6
    assert abs(ref - exact) > 3e-6
