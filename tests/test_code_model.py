"""Host code model (C++ via the C ABI) against the compiled reference (CPU)."""
import os

import numpy as np
import pytest

import paper_2507_03509_b200 as P


def test_spec_examples():
    """SPEC.md code-model examples."""
    h = P.ParityCheckMatrix.from_check_lists(3, [[0, 1], [1, 2]])
    assert (h.n_vars, h.n_checks) == (3, 2) and h.rate() == pytest.approx(1 / 3)
    assert P.active_var_set(h).members.tolist() == [1]
    assert P.syndrome_check(h, [1, 1, 1]) and not P.syndrome_check(h, [1, 1, 0])
    assert P.syndrome_check(h, [0, 0, 0])
    with pytest.raises(P.ValidationError):
        P.syndrome_check(h, [1, 1])
    assert P.vnr_statistic([5, -2, 7], P.ActiveVarSet(np.array([0, 2]))) == 12
    assert P.vnr_statistic([5, -2, 7], P.ActiveVarSet(np.array([], dtype=np.int32))) == 0
    assert P.vnr_should_stop(2.5, 3.0) and not P.vnr_should_stop(3.0, 3.0) and not P.vnr_should_stop(3.1, 3.0)


@pytest.mark.parametrize("n,lists,msg", [
    (0, [[0]], "n_vars must be positive"),
    (3, [[0], [1], [2]], "rate"),
    (3, [], "rate"),
    (3, [[0, 3]], "out of range"),
    (3, [[-1]], "out of range"),
    (3, [[0, 1, 0]], "duplicate edge"),
])
def test_validation_mirrors_reference(ref, n, lists, msg):
    """Same rejections and error class as from_check_lists
    (parity_check_matrix.cpp:10-62): ValidationError (status 3)."""
    with pytest.raises(P.ValidationError, match=msg):
        P.ParityCheckMatrix.from_check_lists(n, lists)
    ptr = np.zeros(len(lists) + 1, dtype=np.int32)
    for c, l in enumerate(lists):
        ptr[c + 1] = ptr[c] + len(l)
    var = np.array([v for l in lists for v in l] or [0], dtype=np.int32)
    import oracle
    with pytest.raises(oracle.OracleError) as e:
        ref.code_from_csr(n, len(lists), ptr, var)
    assert e.value.status == 3 and msg in str(e.value)


def test_alist_roundtrip_with_reference(ref, tmp_path, cfg1_code):
    """Our save_alist is byte-identical to the reference's and both loaders
    agree (alist.cpp:78-202)."""
    ours = tmp_path / "ours.alist"
    theirs = tmp_path / "ref.alist"
    P.save_alist(cfg1_code, str(ours))
    ptr, var = cfg1_code.csr()
    rc = ref.code_from_csr(cfg1_code.n_vars, cfg1_code.n_checks, ptr, var)
    rc.save_alist(str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()
    back = P.load_alist(str(theirs))
    p2, v2 = back.csr()
    assert np.array_equal(p2, ptr) and np.array_equal(v2, var)
    r2 = ref.load_alist(str(ours))
    p3, v3 = r2.csr()
    assert np.array_equal(p3, ptr) and np.array_equal(v3, var)


def test_alist_spec_example(tmp_path):
    f = tmp_path / "h.alist"
    f.write_text("3 2\n2 2\n1 2 1\n2 2\n1\n1 2\n2\n1 2\n2 3\n")
    h = P.load_alist(str(f))
    assert (h.n_vars, h.n_checks) == (3, 2)
    assert [h.check_vars(c).tolist() for c in range(2)] == [[0, 1], [1, 2]]
    g = tmp_path / "g.alist"
    P.save_alist(h, str(g))
    assert g.read_text() == "3 2\n2 2\n1 2 1\n2 2\n1\n1 2\n2\n1 2\n2 3\n"


@pytest.mark.parametrize("text,msg", [
    ("3 2\n2 2\n1 2 1\n2 2\n1\n1 2\n2\n1 2\n2 4\n", "line 9: index 4 out of range"),
    ("3 2\n2 2\n1 2 1\n2 2\n1\n1 2\n2\n1 2\n2 2\n", "duplicate edge"),
    ("3 2\n2 2\n1 2 1\n2 2\n1\n1 2\n2\n1 3\n2 3\n", "adjacency mismatch"),
    ("3 x\n", "expected integer"),
    ("3 2\n2 2\n1 2 1\n", "unexpected end of file"),
    ("2 3\n", "n_checks must be smaller"),
])
def test_alist_errors_match_reference(ref, tmp_path, text, msg):
    f = tmp_path / "bad.alist"
    f.write_text(text)
    with pytest.raises(P.ValidationError, match=msg):
        P.load_alist(str(f))
    import oracle
    with pytest.raises(oracle.OracleError) as e:
        ref.load_alist(str(f))
    assert e.value.status == 3 and msg.split(":")[-1].strip() in str(e.value)


def test_alist_missing_file_is_io_error(tmp_path):
    with pytest.raises(P.IoError):
        P.load_alist(str(tmp_path / "nope.alist"))


@pytest.mark.parametrize("base,z,seed", [([[3, 3]], 1024, 1), ([[2, 1]], 4, 7), ([[1, 1]], 1, 0),
                                         ([[1, 2, 0], [0, 1, 3]], 16, 42)])
def test_lift_protograph_equals_reference(ref, base, z, seed):
    ours = P.lift_protograph(base, z, seed)
    theirs = ref.lift_protograph(base, z, seed)
    p1, v1 = ours.csr()
    p2, v2 = theirs.csr()
    assert np.array_equal(p1, p2) and np.array_equal(v1, v2)


def test_lift_protograph_errors():
    with pytest.raises(P.ValidationError, match="lifting factor too small"):
        P.lift_protograph([[2]], 1, 0)
    with pytest.raises(P.ValidationError):
        P.lift_protograph([[1, -1]], 4, 0)


@pytest.mark.parametrize("key", ["cfg1", "cfg3"])
def test_met_generator_structure(key):
    """BASELINE construction: identity block, class counts, no duplicates,
    near-regular check sockets, determinism."""
    w = P.WORKLOADS[key]
    h = w.make_code()
    n, m = w.n_vars, w.n_checks
    n1 = int(np.floor(w.frac_deg1 * n + 0.5))
    deg = h.var_degrees()
    assert (deg[n - n1:] == 1).all()
    ptr, var = h.csr()
    for j in (0, n1 // 2, n1 - 1):
        assert (n - n1 + j) in h.check_vars(m - n1 + j).tolist()
    nhi = n - n1
    counts = [int(np.floor(nhi * p + 0.5)) for p in w.probs[:-1]]
    counts.append(nhi - sum(counts))
    exp = np.repeat(w.degrees, counts)
    assert np.array_equal(deg[:nhi], exp)
    # no duplicate edges, sorted lists
    for c in range(0, m, max(1, m // 500)):
        l = h.check_vars(c)
        assert np.all(np.diff(l) > 0)
    # near-regular high-degree sockets: every check gets floor or ceil of E_hi/M
    hi_per_check = np.add.reduceat((var < nhi).astype(np.int64), ptr[:-1]) * (np.diff(ptr) > 0)
    e_hi = int(exp.sum())
    assert set(np.unique(hi_per_check)).issubset({e_hi // m, e_hi // m + 1})
    h2 = w.make_code()
    assert np.array_equal(h2.csr()[1], var)


def test_met_generator_sizes():
    """Edge counts of SURVEY §8 for the BASELINE configs."""
    assert P.WORKLOADS["cfg1"].make_code().n_edges == 17820
    c2 = P.WORKLOADS["cfg2"].make_code()
    assert (c2.n_vars, c2.n_checks, c2.n_edges, c2.n_active) == (1048576, 943718, 2280654, 262144)


def test_syndrome_packing(cfg1_code):
    rng = np.random.default_rng(0)
    x = rng.integers(0, 2, size=(3, cfg1_code.n_vars), dtype=np.uint8)
    s = cfg1_code.syndrome(x)
    assert s.shape == (3, (cfg1_code.n_checks + 31) // 32)
    for f in range(3):
        assert P.syndrome_check(cfg1_code, x[f], s[f])
        bad = s[f].copy()
        bad[0] ^= 1
        assert not P.syndrome_check(cfg1_code, x[f], bad)
    assert np.array_equal(P.unpack_bits(P.pack_bits(x), cfg1_code.n_vars), x)


@pytest.mark.parametrize("n,rate,f1,degs,probs,k2", [
    (8192, 0.1, 0.70, (2, 3), (0.5, 0.5), 2),
    (8192, 0.1, 0.85, (2, 3), (0.5, 0.5), 3),
    (20000, 0.02, 0.90, (3,), (1.0,), 3),
])
def test_met_core_generator_structure(n, rate, f1, degs, probs, k2):
    """generate_met_core (csrc/code.cpp): degree-1 variables nc.. on the
    extension checks (one each, identity), every extension check holds
    exactly k2 core variables, core checks hold only core variables, core
    type-1 degree classes in proportion, type-2 degrees within 1 of each
    other, no duplicate edges, deterministic for a seed."""
    m = int(n * (1 - rate) + 0.5)
    n1 = int(f1 * n + 0.5)
    nc, mc = n - n1, m - n1
    code = P.generate_met_core(n, m, n1, degs, probs, k2, 99)
    ptr, var = code.csr()
    assert (code.n_vars, code.n_checks) == (n, m)
    vdeg = code.var_degrees()
    assert np.all(vdeg[nc:] == 1)
    t1 = np.zeros(nc, dtype=np.int64)
    t2 = np.zeros(nc, dtype=np.int64)
    for c in range(m):
        vs = var[ptr[c]:ptr[c + 1]]
        assert len(set(vs.tolist())) == len(vs)
        if c < mc:
            assert np.all(vs < nc)
            np.add.at(t1, vs, 1)
        else:
            core = vs[vs < nc]
            assert len(core) == k2 and vs[-1] == nc + (c - mc) and len(vs) == k2 + 1
            np.add.at(t2, core, 1)
    counts = np.bincount(t1, minlength=max(degs) + 1)
    for d, p in zip(degs[:-1], probs[:-1]):
        assert counts[d] == int(np.floor(nc * p + 0.5))
    assert t2.max() - t2.min() <= 1
    again = P.generate_met_core(n, m, n1, degs, probs, k2, 99)
    assert np.array_equal(again.csr()[1], var) and np.array_equal(again.csr()[0], ptr)
    other = P.generate_met_core(n, m, n1, degs, probs, k2, 100)
    assert not np.array_equal(other.csr()[1], var)


def test_met_core_generator_errors():
    with pytest.raises(P.ValidationError):
        P.generate_met_core(100, 90, 95, (2,), (1.0,), 2, 1)     # n_deg1 >= n_checks
    with pytest.raises(P.ValidationError):
        P.generate_met_core(100, 90, 50, (2, 3), (1.0,), 2, 1)   # misaligned classes
    with pytest.raises(P.ValidationError):
        P.generate_met_core(100, 90, 50, (2,), (1.0,), 0, 1)     # ext_degree 0
