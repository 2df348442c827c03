"""Pins the CPU oracle before it is trusted (CPU only).

* the restatement (oracle.c, ORC_REF_DOUBLE) equals the compiled reference
  bit for bit at s = 0 (bits, iterations, reason, posteriors, q trace);
* in syndrome mode it equals reference(L*(1-2x)) XOR x (sign equivalence);
* both reproduce the known-answer values (tests/golden/kat.json, produced by
  the reference) and the golden frame fixtures;
* SPEC acceptance #3: tree-exact posteriors equal brute-force bitwise MAP.
"""
import itertools
import json

import numpy as np
import pytest

import oracle
from conftest import golden_path

MODES = {"none": (False, False), "pce": (True, False), "vnr": (True, True)}
# 2*atanh(tanh(a/2)*tanh(b/2)) at 50 digits (mpmath)
EXACT = {"sat_30_30": 29.306852819440054690, "sat_12_14": 11.873071988962136593,
         "sat_20_25": 19.993284651510881931}


def kat():
    with open(golden_path("kat.json")) as f:
        return json.load(f)


def test_restatement_kats(orc):
    k = kat()
    o = orc.decode(3, [0, 3], [0, 1, 2], [2.0, 2.0, -0.5], d_max=1, use_pce=False)
    assert o["posteriors"].tolist() == k["spc_posteriors"]  # bit-exact
    assert o["bits"].tolist() == k["spc_bits"] and o["reason"] == k["spc_reason"]
    o = orc.decode(3, [0, 3], [0, 1, 2], [50.0, 50.0, 50.0])
    assert (o["iterations"], o["reason"]) == (k["noiseless_iterations"], k["noiseless_reason"])
    o = orc.decode(2, [0, 1], [0], [-1.0, 3.0], d_max=1, use_pce=False)
    assert o["posteriors"].tolist() == k["deg1_posteriors"]
    for name, l in (("sat_30_30", [30.0, 30.0, 0.0, 1.0]), ("sat_12_14", [12.0, 14.0, 0.0, 1.0]),
                    ("sat_20_25", [20.0, 25.0, 0.0, 1.0])):
        assert orc.decode(4, [0, 3], [0, 1, 2], l, d_max=1, use_pce=False)["posteriors"][2] == k[name]
        # the float phi-domain variant is within 1e-7 of the exact value (mpmath)
        # where float tanh saturates; the reference's double tanh(15) rounding
        # itself costs up to 5.7e-6 relative at the clamp
        f = orc.decode(4, [0, 3], [0, 1, 2], l, d_max=1, use_pce=False, variant=oracle.ORC_PHI_FLOAT)
        assert f["posteriors"][2] == pytest.approx(EXACT[name], rel=1e-7)
        assert f["posteriors"][2] == pytest.approx(k[name], rel=1e-5)
    for key, v in k["snr_for_beta"].items():
        b, r = map(float, key.split(","))
        assert orc.snr_for_beta(b, r) == v
    assert [orc.noise_normal(7, 0, i) for i in range(4)] == k["noise_7_0"]


def test_reference_kats(ref):
    """The compiled reference still reproduces the committed KATs."""
    k = kat()
    spc = ref.code_from_csr(3, 1, [0, 3], [0, 1, 2])
    r = spc.decode_batch(np.array([[2.0, 2.0, -0.5]]), d_max=1, use_pce=False)
    assert r["posteriors"][0].tolist() == k["spc_posteriors"]
    assert ref.noise_normal(7, 0, 4).tolist() == k["noise_7_0"]
    lift = ref.lift_protograph([[3, 3]], 1024, 1)
    assert [lift.n_vars, lift.n_checks, lift.n_edges] == k["lift36_dims"]


def _random_code(rng, n, m, dmin=2, dmax=6):
    lists = [sorted(rng.choice(n, size=int(rng.integers(dmin, dmax + 1)), replace=False).tolist()) for _ in range(m)]
    ptr = np.zeros(m + 1, dtype=np.int32)
    for c, l in enumerate(lists):
        ptr[c + 1] = ptr[c] + len(l)
    return ptr, np.array([v for l in lists for v in l], dtype=np.int32)


@pytest.mark.parametrize("seed", range(6))
def test_restatement_equals_reference_bit_exact(ref, orc, seed):
    rng = np.random.default_rng(seed)
    n, m = 120, 80
    ptr, var = _random_code(rng, n, m, 1, 7)
    rc = ref.code_from_csr(n, m, ptr, var)
    llr = rng.normal(0.6, 1.8, size=(6, n))
    llr[:, :3] = 0.0  # punctured
    for pce, vnr in MODES.values():
        r = rc.decode_batch(llr, d_max=40, use_pce=pce, use_vnr=vnr)
        for b in range(llr.shape[0]):
            o = orc.decode(n, ptr, var, llr[b], d_max=40, use_pce=pce, use_vnr=vnr)
            assert o["iterations"] == r["iterations"][b] and o["reason"] == r["reasons"][b]
            assert np.array_equal(o["bits"], r["bits"][b])
            assert np.array_equal(o["posteriors"], r["posteriors"][b])
            assert np.array_equal(o["q_trace"], r["q_trace"][b][: o["iterations"]])


def test_restatement_equals_reference_cfg1(P, ref, orc, cfg1_code):
    ptr, var = cfg1_code.csr()
    rc = ref.code_from_csr(cfg1_code.n_vars, cfg1_code.n_checks, ptr, var)
    snr = P.snr_for_beta(0.95, cfg1_code.rate())
    llr, x, s = P.sample_frames(cfg1_code, snr, 99, 0, 3)
    leq = (llr * (1 - 2 * x.astype(np.float32))).astype(np.float64)
    for pce, vnr in MODES.values():
        r = rc.decode_batch(leq, d_max=60, use_pce=pce, use_vnr=vnr, threads=3)
        for b in range(3):
            o = orc.decode(cfg1_code.n_vars, ptr, var, leq[b], d_max=60, use_pce=pce, use_vnr=vnr)
            assert o["iterations"] == r["iterations"][b]
            assert np.array_equal(o["posteriors"], r["posteriors"][b])
            # syndrome-mode restatement: sign equivalence
            if not vnr:
                so = orc.decode(cfg1_code.n_vars, ptr, var, llr[b].astype(np.float64), syndrome=s[b], d_max=60,
                                use_pce=pce, use_vnr=vnr)
                assert so["iterations"] == r["iterations"][b]
                assert np.array_equal(so["bits"] ^ x[b], r["bits"][b])
                assert np.array_equal(so["posteriors"] * (1 - 2.0 * x[b]), r["posteriors"][b])


def test_restatement_matches_golden_fixtures(orc):
    for name in ("cfg1_reference.npz", "lift36_reference.npz"):
        z = np.load(golden_path(name))
        n = int(z["n_vars"])
        for mode, (pce, vnr) in MODES.items():
            bits = np.unpackbits(z[f"{mode}_bits"], axis=1)[:, :n]
            for b in range(z["llr_eq"].shape[0]):
                o = orc.decode(n, z["check_ptr"], z["check_vars"], z["llr_eq"][b].astype(np.float64),
                               d_max=int(z["d_max"]), use_pce=pce, use_vnr=vnr)
                assert o["iterations"] == z[f"{mode}_iterations"][b], (name, mode, b)
                assert o["reason"] == z[f"{mode}_reasons"][b]
                assert np.array_equal(o["bits"], bits[b])
                assert np.array_equal(o["posteriors"][:64], z[f"{mode}_posteriors64_head"][b])
                assert np.array_equal(o["posteriors"].astype(np.float32), z[f"{mode}_posteriors"][b])


@pytest.mark.parametrize("variant", [oracle.ORC_PHI_FLOAT, oracle.ORC_T_FLOAT])
def test_phi_float_variant_tracks_reference(P, ref, orc, cfg1_code, variant):
    """The GPU algorithm (float; phi domain, and the shipped t domain)
    restated on the CPU stays within the parity tolerance of the reference on
    config-1 frames."""
    ptr, var = cfg1_code.csr()
    snr = P.snr_for_beta(0.95, cfg1_code.rate())
    llr, x, s = P.sample_frames(cfg1_code, snr, 5, 0, 2)
    leq = (llr * (1 - 2 * x.astype(np.float32))).astype(np.float64)
    rc = ref.code_from_csr(cfg1_code.n_vars, cfg1_code.n_checks, ptr, var)
    r = rc.decode_batch(leq, d_max=200, use_pce=True, use_vnr=True, threads=2)
    for b in range(2):
        o = orc.decode(cfg1_code.n_vars, ptr, var, leq[b], d_max=200, use_pce=True, use_vnr=True,
                       variant=variant)
        assert o["iterations"] == r["iterations"][b]
        assert np.array_equal(o["bits"], r["bits"][b])
        np.testing.assert_allclose(o["posteriors"], r["posteriors"][b], rtol=1e-4, atol=1e-4)


def _map_marginals(n, lists, llr):
    """Exact bitwise MAP LLRs by enumerating all codewords."""
    words = np.array(list(itertools.product([0, 1], repeat=n)), dtype=np.int64)
    ok = np.ones(len(words), dtype=bool)
    for l in lists:
        ok &= (words[:, l].sum(axis=1) % 2) == 0
    cw = words[ok]
    logp = (0.5 * (1 - 2 * cw) * llr[None, :]).sum(axis=1)
    out = np.zeros(n)
    for i in range(n):
        a = np.logaddexp.reduce(logp[cw[:, i] == 0])
        b = np.logaddexp.reduce(logp[cw[:, i] == 1])
        out[i] = a - b
    return out


def _random_tree(rng, n):
    """Cycle-free Tanner graph: checks attach fresh variables to one old one."""
    lists, used = [], [0]
    nxt = 1
    while nxt < n:
        k = int(min(rng.integers(1, 3), n - nxt))
        anchor = int(rng.choice(used))
        l = sorted([anchor] + list(range(nxt, nxt + k)))
        lists.append(l)
        used += list(range(nxt, nxt + k))
        nxt += k
    return lists


@pytest.mark.parametrize("seed", range(20))
def test_tree_exactness_vs_map(orc, seed):
    """SPEC acceptance #3: on >= 20 random cycle-free codes (N <= 12) the
    posteriors after diameter-many iterations equal bitwise MAP to 1e-9
    (clamp disabled by a huge bound)."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(5, 13))
    lists = _random_tree(rng, n)
    if len(lists) >= n:
        pytest.skip("degenerate tree")
    ptr = np.zeros(len(lists) + 1, dtype=np.int32)
    for c, l in enumerate(lists):
        ptr[c + 1] = ptr[c] + len(l)
    var = np.array([v for l in lists for v in l], dtype=np.int32)
    llr = rng.normal(0.5, 1.5, size=n)
    o = orc.decode(n, ptr, var, llr, d_max=2 * n, use_pce=False, use_vnr=False, msg_clamp=1e300)
    np.testing.assert_allclose(o["posteriors"], _map_marginals(n, lists, llr), atol=1e-9, rtol=0)
