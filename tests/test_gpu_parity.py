"""GPU parity: the CUDA decoder (through the C ABI) against the compiled
reference decoder (oracle/_ref) or, where the reference is absent, the
committed golden fixtures it produced (tests/golden/).

Bar (BASELINE.json north star): identical hard decisions, termination
iteration and stop reason on every frame that is not a tie (tests/_parity.py),
posteriors within 1e-4 relative."""
import os

import numpy as np
import pytest

from _parity import compare, ref_ties
from conftest import golden_path

pytestmark = pytest.mark.gpu

ET_MODES = {"none": (False, False), "pce": (True, False), "vnr": (True, True)}


@pytest.fixture(scope="module")
def dec1(P, cfg1_code):
    return P.BatchDecoder(cfg1_code, max_slots=64)


def _refcode(ref, code):
    ptr, var = code.csr()
    return ref.code_from_csr(code.n_vars, code.n_checks, ptr, var)


# ---------------------------------------------------------------- KATs --
def test_kat_single_parity_check(P):
    """SPEC.md:140 / SURVEY App. B: posterior of bit 2 = -0.5 + 2 atanh(tanh(1)^2)."""
    code = P.ParityCheckMatrix.from_check_lists(3, [[0, 1, 2]])
    out = P.BpDecoder(code).decode([2.0, 2.0, -0.5], None, P.DecodeConfig(d_max=1, use_pce=False))
    np.testing.assert_allclose(out.posteriors, [1.6225235436902028, 1.6225235436902028, 0.82500274735786427],
                               rtol=2e-6)
    assert list(out.bits) == [0, 0, 0]
    assert out.reason == P.StopReason.kMaxIterations and out.iterations == 1 and len(out.q_trace) == 1


def test_kat_noiseless_terminates_at_one(P):
    code = P.ParityCheckMatrix.from_check_lists(3, [[0, 1, 2]])
    out = P.BpDecoder(code).decode([50.0, 50.0, 50.0], None, P.DecodeConfig())
    assert out.iterations == 1 and out.reason == P.StopReason.kSyndromeSatisfied and out.converged()


def test_kat_degree1_check_clamps(P):
    """from_check_lists(2, {{0}}), LLR (-1, 3) -> posterior0 = 29."""
    code = P.ParityCheckMatrix.from_check_lists(2, [[0]])
    out = P.BpDecoder(code).decode([-1.0, 3.0], None, P.DecodeConfig(d_max=1, use_pce=False))
    assert out.posteriors[0] == pytest.approx(29.0, abs=0)
    assert out.posteriors[1] == 3.0


def test_kat_saturated_inputs(P):
    """two inputs at the clamp (float tanh would give 30).  Exact
    values from mpmath; the reference's double tanh-domain is itself off by
    5.7e-6 relative at (30, 30) (29.306686), so the GPU is held to the exact
    value at 1e-6 and to the reference at 1e-5."""
    code = P.ParityCheckMatrix.from_check_lists(4, [[0, 1, 2]])
    cases = [((30.0, 30.0), 29.306852819440055, 29.306686431115114),
             ((12.0, 14.0), 11.873071988962137, 11.87307198896398),
             ((20.0, 25.0), 19.993284651510882, 19.993284641387053)]
    for (a, b), exact, refv in cases:
        out = P.BpDecoder(code).decode([a, b, 0.0, 1.0], None, P.DecodeConfig(d_max=1, use_pce=False))
        assert out.posteriors[2] == pytest.approx(exact, rel=1e-6)
        assert out.posteriors[2] == pytest.approx(refv, rel=1e-5)


# ------------------------------------------------- config 1 vs reference --
def _cfg1_frames(P, code, frames=16, beta=0.95, seed=None):
    snr = P.snr_for_beta(beta, code.rate())
    return P.sample_frames(code, snr, P.FRAME_SEED if seed is None else seed, 0, frames)


@pytest.mark.parametrize("mode", list(ET_MODES))
def test_cfg1_all_zero_equivalent_vs_reference(P, ref, cfg1_code, dec1, mode):
    """BASELINE config 1 (16 frames, D_max=200), the reference's own semantics:
    L' = L*(1-2x), s = 0, q = raw sum (decoder.cpp:32-36)."""
    pce, vnr = ET_MODES[mode]
    llr, x, s = _cfg1_frames(P, cfg1_code)
    leq = (llr * (1 - 2 * x.astype(np.float32))).astype(np.float32)
    rc = _refcode(ref, cfg1_code)
    r, tie = ref_ties(rc, leq, d_max=200, use_pce=pce, use_vnr=vnr, threads=8)
    g = dec1.decode_batch(leq, P.DecodeConfig(d_max=200, use_pce=pce, use_vnr=vnr), want_posteriors=True,
                          want_q_trace=True)
    summary = compare(g, r, tie, label=f"cfg1 {mode}")
    # q trace tracks the reference's double q on the frames compared
    for f in np.nonzero(~tie)[0]:
        k = g.iterations[f]
        np.testing.assert_allclose(g.q_trace[f, :k], r["q_trace"][f, :k], rtol=1e-4, atol=1e-2)
    print(summary)


@pytest.mark.parametrize("mode", ["none", "pce"])
def test_cfg1_syndrome_mode_vs_reference(P, ref, cfg1_code, dec1, mode):
    """True syndrome mode (L, s = Hx) equals reference(L*(1-2x)) XOR x
    (sign equivalence) for ET none / PCE."""
    pce, vnr = ET_MODES[mode]
    llr, x, s = _cfg1_frames(P, cfg1_code)
    leq = (llr * (1 - 2 * x.astype(np.float32))).astype(np.float32)
    rc = _refcode(ref, cfg1_code)
    r, tie = ref_ties(rc, leq, d_max=200, use_pce=pce, use_vnr=vnr, threads=8)
    g = dec1.decode_batch(llr, P.DecodeConfig(d_max=200, use_pce=pce, use_vnr=vnr), syndrome=s,
                          want_posteriors=True)
    g.bits = g.bits ^ x
    g.posteriors = g.posteriors * (1 - 2 * x.astype(np.float32))
    compare(g, r, tie, label=f"cfg1 syndrome {mode}")


def test_syndrome_mode_equivalence_bit_exact(P, cfg1_code, dec1):
    """decode(L, Hx) == decode(L*(1-2x), 0) XOR x bit for bit on the GPU —
    including VNR with the x-free q = sum|l| (the kernel arithmetic is exactly
    sign-symmetric)."""
    llr, x, s = _cfg1_frames(P, cfg1_code, frames=40, beta=0.9)
    leq = (llr * (1 - 2 * x.astype(np.float32))).astype(np.float32)
    for pce, vnr in ET_MODES.values():
        cfg = P.DecodeConfig(d_max=200, use_pce=pce, use_vnr=vnr, q_mode=P.decoder.Q_ABS)
        a = dec1.decode_batch(llr, cfg, syndrome=s, want_posteriors=True)
        b = dec1.decode_batch(leq, cfg, want_posteriors=True)
        assert np.array_equal(a.iterations, b.iterations)
        assert np.array_equal(a.reasons, b.reasons)
        assert np.array_equal(a.bits ^ x, b.bits)
        assert np.array_equal(a.posteriors * (1 - 2 * x.astype(np.float32)), b.posteriors)


def test_cfg1_golden_fixture(P, cfg1_code, dec1):
    """Same comparison against the committed reference outputs (usable where
    the reference library is absent)."""
    path = golden_path("cfg1_reference.npz")
    if not os.path.exists(path):
        pytest.skip("golden fixture not generated")
    z = np.load(path)
    for mode, (pce, vnr) in ET_MODES.items():
        leq = z["llr_eq"]
        g = dec1.decode_batch(leq, P.DecodeConfig(d_max=int(z["d_max"]), use_pce=pce, use_vnr=vnr),
                              want_posteriors=True)
        bits = np.unpackbits(z[f"{mode}_bits"], axis=1)[:, :cfg1_code.n_vars]
        r = {"bits": bits, "iterations": z[f"{mode}_iterations"], "reasons": z[f"{mode}_reasons"],
             "posteriors": z[f"{mode}_posteriors"], "drift": z[f"{mode}_drift"]}
        compare(g, r, z[f"{mode}_tie"], label=f"golden {mode}")


# ----------------------------------------------- (3,6) lift, converging --
@pytest.mark.parametrize("beta", [0.6, 0.7, 0.8])
@pytest.mark.parametrize("mode", list(ET_MODES))
def test_lift36_vs_reference(P, ref, lift36, beta, mode):
    """The reference's (3,6) N=2048 code: converging and
    non-converging frames; chaotic frames are ties by the reference's own
    one-ulp sensitivity."""
    pce, vnr = ET_MODES[mode]
    dec = P.BatchDecoder(lift36, max_slots=64)
    snr = P.snr_for_beta(beta, lift36.rate())
    llr, _, _ = P.sample_frames(lift36, snr, 77, 0, 64, all_zero=True)
    rc = _refcode(ref, lift36)
    r, tie = ref_ties(rc, llr, d_max=200, use_pce=pce, use_vnr=vnr, threads=8)
    g = dec.decode_batch(llr, P.DecodeConfig(d_max=200, use_pce=pce, use_vnr=vnr), want_posteriors=True)
    print(compare(g, r, tie, min_nontie_frac=0.2, failed_decode_slack=0.05, label=f"lift36 beta={beta} {mode}"))


# --------------------------------------------------------- edge cases --
def test_punctured_zero_llrs(P, ref, lift36):
    """LLR = 0 entries (puncturing, decoder.hpp:59-61) through the phi(0)=inf path."""
    dec = P.BatchDecoder(lift36, max_slots=32)
    snr = P.snr_for_beta(0.5, lift36.rate())
    llr, _, _ = P.sample_frames(lift36, snr, 5, 0, 8, all_zero=True)
    rng = np.random.default_rng(1)
    llr[:, rng.choice(lift36.n_vars, 200, replace=False)] = 0.0
    rc = _refcode(ref, lift36)
    r, tie = ref_ties(rc, llr, d_max=100, use_pce=True, use_vnr=False, threads=8)
    g = dec.decode_batch(llr, P.DecodeConfig(d_max=100), want_posteriors=True)
    compare(g, r, tie, label="punctured")


def test_irregular_edge_cases(P, ref):
    """Degree-0 checks, degree-1 checks, degree-0 variables, a high-degree
    check (generic kernel path), LLR beyond the clamp."""
    rng = np.random.default_rng(3)
    n = 300
    lists = []
    for c in range(200):
        r = c % 10
        if r == 0:
            lists.append([])                                  # degree-0 check
        elif r == 1:
            lists.append([int(rng.integers(0, 280))])         # degree-1 check
        else:
            lists.append(sorted(rng.choice(280, size=int(rng.integers(2, 7)), replace=False).tolist()))
    lists[2] = sorted(rng.choice(280, size=40, replace=False).tolist())  # degree 40 -> generic path
    code = P.ParityCheckMatrix.from_check_lists(n, lists)  # vars 280..299 have degree 0
    dec = P.BatchDecoder(code, max_slots=32)
    llr = rng.normal(0.8, 1.5, size=(24, n)).astype(np.float32)
    llr[:, :5] = 45.0   # beyond the clamp: first iteration unclamped, later clamped
    llr[:, 5:8] = -45.0
    rc = _refcode(ref, code)
    for pce, vnr in ET_MODES.values():
        r, tie = ref_ties(rc, llr, d_max=60, use_pce=pce, use_vnr=vnr, threads=8)
        g = dec.decode_batch(llr, P.DecodeConfig(d_max=60, use_pce=pce, use_vnr=vnr), want_posteriors=True)
        compare(g, r, tie, label=f"irregular pce={pce} vnr={vnr}")


def test_high_degree_variables(P, ref):
    """Variable degrees 14 / 20 / 27 (typed variable path, each variable split
    over several batches, tiles padded to degree 16 / 20 / 32), 36 (generic
    path) and mixed-degree boundary tiles, next to degree-3 and degree-1
    variables."""
    rng = np.random.default_rng(11)
    classes = [(3, 100), (14, 128), (20, 128), (27, 64), (36, 64)]
    degs = np.concatenate([np.full(n, d) for d, n in classes])
    n_hi = len(degs)
    m = 1400
    lists = [set() for _ in range(m)]
    for v, d in enumerate(degs):
        for c in rng.choice(m, size=int(d), replace=False):
            lists[int(c)].add(v)
    # one degree-1 variable per check (identity block, as in the BASELINE codes)
    lists = [sorted(c) + [n_hi + j] for j, c in enumerate(lists)]
    code = P.ParityCheckMatrix.from_check_lists(n_hi + m, lists)
    dec = P.BatchDecoder(code, max_slots=32)
    llr = rng.normal(0.9, 1.4, size=(24, code.n_vars)).astype(np.float32)
    rc = _refcode(ref, code)
    for pce, vnr in ET_MODES.values():
        r, tie = ref_ties(rc, llr, d_max=40, use_pce=pce, use_vnr=vnr, threads=8)
        g = dec.decode_batch(llr, P.DecodeConfig(d_max=40, use_pce=pce, use_vnr=vnr), want_posteriors=True)
        compare(g, r, tie, label=f"high-degree pce={pce} vnr={vnr}")


def test_dmax_one_and_batch_shapes(P, ref, cfg1_code):
    """d_max = 1, B = 1, B not a multiple of 32, B > slots (frames stream
    through recycled slots)."""
    rc = _refcode(ref, cfg1_code)
    snr = P.snr_for_beta(0.3, cfg1_code.rate())
    llr, _, _ = P.sample_frames(cfg1_code, snr, 9, 0, 75, all_zero=True)
    dec = P.BatchDecoder(cfg1_code, max_slots=32)
    for d_max, B in [(1, 1), (1, 75), (30, 37), (30, 75)]:
        r, tie = ref_ties(rc, llr[:B], d_max=d_max, use_pce=True, use_vnr=True, threads=8)
        g = dec.decode_batch(llr[:B], P.DecodeConfig(d_max=d_max, use_pce=True, use_vnr=True),
                             want_posteriors=True)
        compare(g, r, tie, label=f"d_max={d_max} B={B}")


def test_packed_bits_and_device_buffers(P, cfg1_code):
    import torch
    dec = P.BatchDecoder(cfg1_code, max_slots=64)
    snr = P.snr_for_beta(0.2, cfg1_code.rate())
    llr, x, s = P.sample_frames(cfg1_code, snr, 21, 0, 40)
    cfg = P.DecodeConfig(d_max=100, use_pce=True, use_vnr=False)
    a = dec.decode_batch(llr, cfg, syndrome=s)
    b = dec.decode_batch(llr, cfg, syndrome=s, packed=True)
    assert np.array_equal(P.unpack_bits(b.bits, cfg1_code.n_vars), a.bits)
    dl = torch.from_numpy(llr).cuda()
    ds = torch.from_numpy(s.view(np.int32)).cuda()
    out = {"iterations": torch.zeros(40, dtype=torch.int32, device="cuda"),
           "reasons": torch.zeros(40, dtype=torch.uint8, device="cuda"),
           "bits": torch.zeros((40, cfg1_code.n_vars), dtype=torch.uint8, device="cuda")}
    c = dec.decode_batch(dl, cfg, syndrome=ds, out=out)
    assert np.array_equal(c.bits.cpu().numpy(), a.bits)
    assert np.array_equal(c.iterations.cpu().numpy(), a.iterations)
    # success => H bits == s
    for f in range(40):
        if a.reasons[f] == 0:
            assert P.syndrome_check(cfg1_code, a.bits[f], s[f])


def test_staged_host_inputs(P, cfg1_code):
    """bpdec_decoder_stage_inputs: a staged host batch decodes exactly like an
    unstaged one; staging overlaps the next batch's upload; a replaced stage
    falls back to the normal copy; device inputs are rejected."""
    import torch
    dec = P.BatchDecoder(cfg1_code, max_slots=32)
    snr = P.snr_for_beta(0.95, cfg1_code.rate())
    cfg = P.DecodeConfig(d_max=200, use_pce=True, use_vnr=True, q_mode=P.decoder.Q_ABS)
    batches = []
    for k in range(4):
        llr, x, s = P.sample_frames(cfg1_code, snr, 41, 40 * k, 40)
        hl = torch.from_numpy(llr).pin_memory()
        hs = torch.from_numpy(s.view(np.int32)).pin_memory()
        batches.append((hl, hs, dec.decode_batch(llr, cfg, syndrome=s, want_posteriors=True)))
    # pipelined: stage k+1 before decoding k
    dec.stage_inputs(batches[0][0], batches[0][1])
    for k in range(4):
        if k + 1 < 4:
            dec.stage_inputs(batches[k + 1][0], batches[k + 1][1])
        hl, hs, want = batches[k]
        g = dec.decode_batch(hl, cfg, syndrome=hs, want_posteriors=True)
        assert np.array_equal(g.bits, want.bits) and np.array_equal(g.iterations, want.iterations)
        assert np.array_equal(g.posteriors, want.posteriors)
    # three stages: the oldest is replaced, its decode copies again
    for k in range(3):
        dec.stage_inputs(batches[k][0], batches[k][1])
    for k in range(3):
        g = dec.decode_batch(batches[k][0], cfg, syndrome=batches[k][1])
        assert np.array_equal(g.bits, batches[k][2].bits)
    with pytest.raises(P.ValidationError):
        dec.stage_inputs(batches[0][0].cuda(), None)


def test_failed_construction_is_clean(P, cfg1_code):
    """A bad device index or an impossible slot count fails with the right
    error class and releases what it allocated; decoders still work after."""
    with pytest.raises(P.ConfigError):
        P.BatchDecoder(cfg1_code, device=99, max_slots=32)
    with pytest.raises(P.ValidationError):
        P.BatchDecoder(cfg1_code, max_slots=0)
    big = P.generate_met(1 << 20, 943718, 0.75, (3, 6, 12), (0.5, 0.3, 0.2), 7)
    for _ in range(3):  # ~15 GB per attempt would exhaust the GPU if leaked
        with pytest.raises((P.decoder.BpdecOomError, P.ValidationError)):
            P.BatchDecoder(big, max_slots=32768)
    dec = P.BatchDecoder(cfg1_code, max_slots=32)
    llr, _, _ = P.sample_frames(cfg1_code, P.snr_for_beta(0.9, cfg1_code.rate()), 3, 0, 4, all_zero=True)
    assert dec.decode_batch(llr, P.DecodeConfig(d_max=10)).iterations.shape == (4,)


def test_nonfinite_llr_rejected(P, cfg1_code):
    dec = P.BatchDecoder(cfg1_code, max_slots=32)
    llr = np.zeros((2, cfg1_code.n_vars), dtype=np.float32)
    llr[1, 17] = np.nan
    with pytest.raises(P.ValidationError):
        dec.decode_batch(llr, P.DecodeConfig())
    with pytest.raises(P.ValidationError):
        dec.decode_batch(llr[:1], P.DecodeConfig(d_max=0))


# ------------------------------------------- determinism / sharding --
def test_determinism_and_slot_invariance(P, cfg1_code):
    """Per-frame outputs do not depend on run, slot count, batch composition
    or frame order — the property that makes 1/2/4/8-GPU sharding exact."""
    snr = P.snr_for_beta(0.95, cfg1_code.rate())
    llr, x, s = P.sample_frames(cfg1_code, snr, 31, 0, 96)
    cfg = P.DecodeConfig(d_max=200, use_pce=True, use_vnr=True, q_mode=P.decoder.Q_ABS)
    ref = P.BatchDecoder(cfg1_code, max_slots=96).decode_batch(llr, cfg, syndrome=s, want_posteriors=True,
                                                               want_q_trace=True)
    for slots in (32, 64):
        d = P.BatchDecoder(cfg1_code, max_slots=slots)
        for order in (np.arange(96), np.arange(96)[::-1]):
            g = d.decode_batch(llr[order], cfg, syndrome=s[order], want_posteriors=True, want_q_trace=True)
            assert np.array_equal(g.iterations, ref.iterations[order])
            assert np.array_equal(g.bits, ref.bits[order])
            assert np.array_equal(g.posteriors, ref.posteriors[order])
            assert np.array_equal(g.q_trace, ref.q_trace[order], equal_nan=True)
    # shards: frames [0,48) and [48,96) decoded separately == together
    d = P.BatchDecoder(cfg1_code, max_slots=64)
    parts = [d.decode_batch(llr[a:b], cfg, syndrome=s[a:b], want_posteriors=True) for a, b in ((0, 48), (48, 96))]
    assert np.array_equal(np.concatenate([p.bits for p in parts]), ref.bits)
    assert np.array_equal(np.concatenate([p.iterations for p in parts]), ref.iterations)


def test_streaming_turnover_paths(P, cfg1_code):
    """Frames streaming through few slots (refills of 1..32 lanes per group,
    sparse and dense refill paths, independent extraction) give the same
    per-frame results as one frame per slot, with and without posteriors."""
    snr = P.snr_for_beta(0.95, cfg1_code.rate())
    llr, x, s = P.sample_frames(cfg1_code, snr, 51, 0, 200)
    cfg = P.DecodeConfig(d_max=120, use_pce=True, use_vnr=True, q_mode=P.decoder.Q_ABS)
    ref = P.BatchDecoder(cfg1_code, max_slots=224).decode_batch(llr, cfg, syndrome=s, want_posteriors=True)
    for slots in (32, 96):
        d = P.BatchDecoder(cfg1_code, max_slots=slots)
        for packed in (False, True):
            g = d.decode_batch(llr, cfg, syndrome=s, packed=packed)
            bits = P.unpack_bits(g.bits, cfg1_code.n_vars) if packed else g.bits
            assert np.array_equal(bits, ref.bits), (slots, packed)
            assert np.array_equal(g.iterations, ref.iterations) and np.array_equal(g.reasons, ref.reasons)
        g = d.decode_batch(llr, cfg, syndrome=s, want_posteriors=True)
        assert np.array_equal(g.posteriors, ref.posteriors)


def test_device_generator_matches_host(P, cfg1_code):
    import torch
    dec = P.BatchDecoder(cfg1_code, max_slots=32)
    snr = P.snr_for_beta(0.95, cfg1_code.rate())
    llr, x, s = P.sample_frames(cfg1_code, snr, 123, 5, 8)
    dl = torch.empty((8, cfg1_code.n_vars), dtype=torch.float32, device="cuda")
    ds = torch.empty((8, (cfg1_code.n_checks + 31) // 32), dtype=torch.int32, device="cuda")
    dx = torch.empty((8, (cfg1_code.n_vars + 31) // 32), dtype=torch.int32, device="cuda")
    dec.sample_frames_device(snr, 123, 5, 8, dl, ds, dx)
    gl = dl.cpu().numpy()
    # device libm may differ from glibc by an ulp in rare draws
    mism = np.abs(gl.view(np.int32).astype(np.int64) - llr.view(np.int32).astype(np.int64))
    assert mism.max() <= 1 and (mism > 0).mean() < 1e-3
    assert np.array_equal(ds.cpu().numpy().view(np.uint32), s)
    assert np.array_equal(P.unpack_bits(dx.cpu().numpy().view(np.uint32), cfg1_code.n_vars), x)


def test_tail_compaction_is_transparent(P, cfg1_code):
    """Group compaction (queue drained, live frames fit in fewer 32-slot
    groups) moves frames between slots mid-decode; every per-frame output
    must be bit-identical to decoding each frame alone."""
    snr = P.snr_for_beta(0.95, cfg1_code.rate())
    llr, x, s = P.sample_frames(cfg1_code, snr, 4242, 0, 128)
    cfg = P.DecodeConfig(d_max=200, use_pce=True, use_vnr=True, q_mode=P.decoder.Q_ABS)
    big = P.BatchDecoder(cfg1_code, max_slots=128)  # 4 groups, compaction as frames stop
    r = big.decode_batch(llr, cfg, syndrome=s, want_posteriors=True, want_q_trace=True)
    assert len(set(r.iterations.tolist())) > 5  # stop times spread: the tail compacts
    one = P.BatchDecoder(cfg1_code, max_slots=32)
    for f in range(0, 128, 9):
        o = one.decode_batch(llr[f:f + 1], cfg, syndrome=s[f:f + 1], want_posteriors=True, want_q_trace=True)
        assert o.iterations[0] == r.iterations[f] and o.reasons[0] == r.reasons[f]
        assert np.array_equal(o.bits[0], r.bits[f])
        assert np.array_equal(o.posteriors[0], r.posteriors[f])
        assert np.array_equal(o.q_trace[0], r.q_trace[f], equal_nan=True)


def _decode_all(dec, llr, s, cfg):
    return dec.decode_batch(llr, cfg, syndrome=s, want_posteriors=True, want_q_trace=True)


def _assert_same(a, b, idx=None):
    sel = slice(None) if idx is None else idx
    assert np.array_equal(a.iterations, b.iterations[sel]) and np.array_equal(a.reasons, b.reasons[sel])
    assert np.array_equal(a.bits, b.bits[sel])
    assert np.array_equal(a.posteriors, b.posteriors[sel])
    assert np.array_equal(a.q_trace, b.q_trace[sel], equal_nan=True)


def _with_degree1_checks(P, code, n01=48, n10=24):
    """The config-1 code plus n01 checks holding one new degree-1 variable
    each (type (0,1)) and n10 single-edge checks on existing degree>=2
    variables (type (1,0)) — check types k_check skips after a frame's first
    iteration."""
    ptr, var = code.csr()
    lists = [list(var[ptr[c]:ptr[c + 1]]) for c in range(code.n_checks)]
    n = code.n_vars
    lists += [[n + i] for i in range(n01)]
    hi = np.nonzero(code.var_degrees() >= 2)[0]
    lists += [[int(v)] for v in hi[:: max(1, len(hi) // n10)][:n10]]
    return P.ParityCheckMatrix.from_check_lists(n + n01, lists)


def _highdeg_code(P):
    """Check degree <= 3 (sockets dealt round-robin, as the BASELINE
    generator does) with variables of degree 3, 14, 20, 27 and 36: split
    variable batches (wide) / unsplit (narrow), tiles padded to 16 / 20 /
    32, and the generic variable path (degree 36), plus one degree-1
    variable per check."""
    classes = [(3, 600), (14, 40), (20, 40), (27, 20), (36, 20)]
    m = 3000
    lists = [[] for _ in range(m)]
    k = 0
    v = 0
    for d, n in classes:
        for _ in range(n):
            for _ in range(d):
                lists[k % m].append(v)
                k += 1
            v += 1
    lists = [sorted(c) + [v + j] for j, c in enumerate(lists)]
    return P.ParityCheckMatrix.from_check_lists(v + m, lists)


@pytest.mark.parametrize("kind", ["cfg1", "deg1checks", "highdeg"])
def test_narrow_tail_bit_exact(P, cfg1_code, kind):
    """Narrow tail groups (the only live group re-laid out with 16 / 8 lanes
    per row, lane-folded check and variable passes) and group compaction
    move frames mid-decode.  Every per-frame output — bits, iterations,
    reasons, posteriors and the q trace — must equal (a) the all-wide decode
    (BPDEC_NO_NARROW=1) and (b) decoding the frame alone in a one-group
    decoder (no moves).  "deg1checks" adds degree-1-only checks, whose
    words k_check recomputes only in a frame's first iteration or after
    frames moved."""
    if kind == "cfg1":
        code = cfg1_code
    elif kind == "deg1checks":
        code = _with_degree1_checks(P, cfg1_code)
        assert (code.check_degrees() == 1).sum() == 48 + 24
    else:
        code = _highdeg_code(P)
        assert code.check_degrees().max() <= 4 and code.var_degrees().max() == 36
    # VNR: stop times spread at any beta; PCE alone: in the converging regime
    for pce, vnr, blo, bhi in ((True, True, 0.2, 1.0), (True, False, 0.05, 0.35)):
        llr, x, s, _ = P.sample_frames_beta(code, blo, bhi, 808, 0, 96)
        if kind == "highdeg":  # a low-rate-like channel where the code's own SNR map does not apply
            rng = np.random.default_rng(5)
            mu = rng.uniform(0.2, 1.6, size=(96, 1)) if not vnr else rng.uniform(0.05, 0.6, size=(96, 1))
            llr = (mu + rng.normal(0.0, 1.0, size=(96, code.n_vars)) * np.sqrt(2 * mu)).astype(np.float32)
            s = np.zeros_like(s)
        cfg = P.DecodeConfig(d_max=150, use_pce=pce, use_vnr=vnr, q_mode=P.decoder.Q_ABS)
        r = _decode_all(P.BatchDecoder(code, max_slots=96), llr, s, cfg)  # 3 groups: compaction, narrowing
        assert len(set(r.iterations.tolist())) > 4, "stop times must spread for the tail to form"
        os.environ["BPDEC_NO_NARROW"] = "1"
        try:
            w = _decode_all(P.BatchDecoder(code, max_slots=96), llr, s, cfg)
        finally:
            del os.environ["BPDEC_NO_NARROW"]
        _assert_same(w, r)
        one = P.BatchDecoder(code, max_slots=32)
        for f in list(range(0, 96, 7)) + [int(np.argmax(r.iterations))]:
            _assert_same(_decode_all(one, llr[f:f + 1], s[f:f + 1], cfg), r, slice(f, f + 1))

# BASELINE configurations at full size: tests/test_gpu_baseline.py
