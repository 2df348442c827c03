"""TEST INFRASTRUCTURE — ctypes access to the CPU checkers.

* ``Reference``: the unmodified reference library (oracle/_ref/libetdec_ref.so,
  built from /root/reference/proj/core/src by oracle/Makefile + ref_shim.cpp).
* ``Restatement``: the plain-C restatement (oracle/_build/liboracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product
(paper_2507_03509_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libetdec_ref.so")
ORC_LIB = os.path.join(HERE, "_build", "liboracle.so")

ORC_REF_DOUBLE, ORC_PHI_FLOAT, ORC_T_FLOAT = 0, 1, 2
# the float32 variant of the shipped CUDA kernels (phi.cuh: t domain)
ORC_GPU_FLOAT = ORC_T_FLOAT


def _p(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


def build() -> None:
    """Builds the checkers in place (make -C oracle)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class OracleError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"status {status}: {msg}")
        self.status = status


class Reference:
    """The compiled reference (etdec_core), run in its run_trials threading
    pattern (one BpDecoder per std::thread, frames strided)."""

    def __init__(self):
        if not os.path.exists(REF_LIB):
            raise FileNotFoundError(f"{REF_LIB} missing (build with `make -C oracle` where /root/reference exists)")
        L = C.CDLL(REF_LIB)
        vp, i32, u8, f64 = C.c_void_p, C.c_int32, C.c_uint8, C.c_double
        L.etref_code_create.restype = vp
        L.etref_code_create.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.etref_code_load_alist.restype = vp
        L.etref_code_load_alist.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.etref_code_save_alist.argtypes = [vp, C.c_char_p]
        L.etref_lift_protograph.restype = vp
        L.etref_lift_protograph.argtypes = [C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, C.c_uint64,
                                            C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.etref_code_destroy.argtypes = [vp]
        L.etref_code_dims.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.etref_code_csr.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.etref_decode_batch.argtypes = [vp, C.c_int, C.POINTER(f64), C.c_int, C.c_int, C.c_int, f64, C.c_int,
                                         C.POINTER(u8), C.POINTER(i32), C.POINTER(u8), C.POINTER(f64),
                                         C.POINTER(f64), C.c_char_p, C.c_int]
        L.etref_decode_observed.argtypes = [vp, C.POINTER(f64), C.c_int, C.c_int, C.c_int, f64, C.POINTER(i32),
                                            C.POINTER(u8), C.POINTER(u8), C.POINTER(f64), C.POINTER(i32)]
        L.etref_decode_observed_post.argtypes = [vp, C.POINTER(f64), C.c_int, C.c_int, C.c_int, f64, C.POINTER(i32),
                                                 C.POINTER(u8), C.POINTER(u8), C.POINTER(f64), C.POINTER(f64),
                                                 C.POINTER(i32)]
        L.etref_syndrome_check.argtypes = [vp, C.POINTER(u8), C.c_int]
        L.etref_snr_for_beta.restype = f64
        L.etref_snr_for_beta.argtypes = [f64, f64]
        L.etref_noise_normal.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.POINTER(f64)]
        L.etref_sample_block.argtypes = [f64, C.c_int, C.c_uint64, C.c_uint64, C.POINTER(f64)]
        L.etref_apply_puncture.argtypes = [vp, f64, C.c_uint64, C.POINTER(C.c_int), C.POINTER(f64)]
        L.etref_run_trials.argtypes = [vp, C.POINTER(C.c_int), C.c_int, f64, C.c_int, C.c_int, C.c_int, f64, C.c_long,
                                       C.c_long, C.c_uint64, C.c_int, C.POINTER(C.c_int64), C.POINTER(f64),
                                       C.POINTER(C.c_int64), C.c_int]
        L.etref_vnr_statistic.restype = f64
        L.etref_vnr_statistic.argtypes = [C.POINTER(f64), C.POINTER(C.c_int), C.c_int]
        self.L = L

    # -- codes
    def code_from_csr(self, n_vars, n_checks, check_ptr, check_vars):
        ptr = np.ascontiguousarray(check_ptr, dtype=np.int32)
        var = np.ascontiguousarray(check_vars, dtype=np.int32)
        st = C.c_int()
        err = C.create_string_buffer(512)
        h = self.L.etref_code_create(n_vars, n_checks, _p(ptr, C.c_int), _p(var, C.c_int), C.byref(st), err, 512)
        if not h:
            raise OracleError(st.value, err.value.decode())
        return RefCode(self, h)

    def load_alist(self, path):
        st = C.c_int()
        err = C.create_string_buffer(512)
        h = self.L.etref_code_load_alist(path.encode(), C.byref(st), err, 512)
        if not h:
            raise OracleError(st.value, err.value.decode())
        return RefCode(self, h)

    def lift_protograph(self, base, z, seed):
        b = np.ascontiguousarray(base, dtype=np.int32)
        st = C.c_int()
        err = C.create_string_buffer(512)
        h = self.L.etref_lift_protograph(_p(b, C.c_int), b.shape[0], b.shape[1], z, seed, C.byref(st), err, 512)
        if not h:
            raise OracleError(st.value, err.value.decode())
        return RefCode(self, h)

    def snr_for_beta(self, beta, rate):
        return self.L.etref_snr_for_beta(beta, rate)

    def noise_normal(self, seed, stream, count):
        out = np.zeros(count, dtype=np.float64)
        self.L.etref_noise_normal(seed, stream, count, _p(out, C.c_double))
        return out

    def sample_block(self, snr, n, seed, trial):
        out = np.zeros(n, dtype=np.float64)
        self.L.etref_sample_block(snr, n, seed, trial, _p(out, C.c_double))
        return out


class RefCode:
    def __init__(self, ref: Reference, h):
        self.ref, self.h = ref, h
        n, m, e = C.c_int(), C.c_int(), C.c_int()
        ref.L.etref_code_dims(h, C.byref(n), C.byref(m), C.byref(e))
        self.n_vars, self.n_checks, self.n_edges = n.value, m.value, e.value

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.L.etref_code_destroy(self.h)
            self.h = None

    def csr(self):
        ptr = np.zeros(self.n_checks + 1, dtype=np.int32)
        var = np.zeros(max(self.n_edges, 1), dtype=np.int32)
        self.ref.L.etref_code_csr(self.h, _p(ptr, C.c_int), _p(var, C.c_int))
        return ptr, var[: self.n_edges]

    def save_alist(self, path):
        st = self.ref.L.etref_code_save_alist(self.h, path.encode())
        if st:
            raise OracleError(st)

    def syndrome_check(self, bits):
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        r = self.ref.L.etref_syndrome_check(self.h, _p(b, C.c_uint8), b.size)
        if r < 0:
            raise OracleError(-r)
        return bool(r)

    def apply_puncture(self, target_rate, seed):
        out = np.zeros(self.n_vars, dtype=np.int32)
        eff = C.c_double()
        n = self.ref.L.etref_apply_puncture(self.h, target_rate, seed, _p(out, C.c_int), C.byref(eff))
        if n < 0:
            raise OracleError(-n)
        return out[:n], eff.value

    def run_trials(self, beta, punctured=None, d_max=100, use_pce=True, use_vnr=False, msg_clamp=30.0,
                   min_frame_errors=100, max_frames=10000, seed=1, workers=8):
        """The reference's own run_trials (channel.cpp:74-156)."""
        p = np.ascontiguousarray(np.zeros(0) if punctured is None else punctured, dtype=np.int32)
        st = np.zeros(8, dtype=np.int64)
        ds = np.zeros(4, dtype=np.float64)
        hist = np.zeros(d_max + 1, dtype=np.int64)
        r = self.ref.L.etref_run_trials(self.h, _p(p, C.c_int), p.size, beta, d_max, int(use_pce), int(use_vnr),
                                        msg_clamp, min_frame_errors, max_frames, seed, workers, _p(st, C.c_int64),
                                        _p(ds, C.c_double), _p(hist, C.c_int64), hist.size)
        if r:
            raise OracleError(r)
        return dict(frames=int(st[0]), frame_errors=int(st[1]), undetected_errors=int(st[2]),
                    iteration_sum=int(st[3]), stops_syndrome=int(st[4]), stops_vnr=int(st[5]),
                    stops_max_iter=int(st[6]), hit_max_frames=bool(st[7]), fer=ds[0], fer_ci_low=ds[1],
                    fer_ci_high=ds[2], d_bar=ds[3], histogram={int(k): int(v) for k, v in enumerate(hist) if v})

    def decode_batch(self, llr, d_max=100, use_pce=True, use_vnr=False, msg_clamp=30.0, threads=1,
                     want_posteriors=True, want_q_trace=True):
        """Reference decode of every frame of llr [B, N] (double)."""
        llr = np.ascontiguousarray(llr, dtype=np.float64)
        if llr.ndim == 1:
            llr = llr[None, :]
        B, n = llr.shape
        bits = np.zeros((B, n), dtype=np.uint8)
        it = np.zeros(B, dtype=np.int32)
        rs = np.zeros(B, dtype=np.uint8)
        post = np.zeros((B, n), dtype=np.float64) if want_posteriors else None
        qt = np.zeros((B, d_max), dtype=np.float64) if want_q_trace else None
        err = C.create_string_buffer(512)
        st = self.ref.L.etref_decode_batch(self.h, B, _p(llr, C.c_double), d_max, int(use_pce), int(use_vnr),
                                           msg_clamp, threads, _p(bits, C.c_uint8), _p(it, C.c_int32),
                                           _p(rs, C.c_uint8), _p(post, C.c_double), _p(qt, C.c_double), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return dict(bits=bits, iterations=it, reasons=rs, posteriors=post, q_trace=qt)

    def decode_observed(self, llr, d_max=100, use_pce=True, use_vnr=False, msg_clamp=30.0):
        llr = np.ascontiguousarray(llr, dtype=np.float64)
        it, rs, calls = C.c_int32(), C.c_uint8(), C.c_int32()
        ok = np.zeros(d_max, dtype=np.uint8)
        q = np.zeros(d_max, dtype=np.float64)
        st = self.ref.L.etref_decode_observed(self.h, _p(llr, C.c_double), d_max, int(use_pce), int(use_vnr),
                                              msg_clamp, C.byref(it), C.byref(rs), _p(ok, C.c_uint8),
                                              _p(q, C.c_double), C.byref(calls))
        if st:
            raise OracleError(st)
        k = it.value
        return dict(iterations=k, reason=rs.value, syndrome_ok=ok[:k], q=q[:k], calls=calls.value)

    def decode_observed_post(self, llr, d_max=100, use_pce=True, use_vnr=False, msg_clamp=30.0):
        """decode_observed plus the observer's per-iteration posteriors."""
        llr = np.ascontiguousarray(llr, dtype=np.float64)
        n = llr.size
        it, rs, calls = C.c_int32(), C.c_uint8(), C.c_int32()
        ok = np.zeros(d_max, dtype=np.uint8)
        q = np.zeros(d_max, dtype=np.float64)
        post = np.zeros((d_max, n), dtype=np.float64)
        st = self.ref.L.etref_decode_observed_post(self.h, _p(llr, C.c_double), d_max, int(use_pce), int(use_vnr),
                                                   msg_clamp, C.byref(it), C.byref(rs), _p(ok, C.c_uint8),
                                                   _p(q, C.c_double), _p(post, C.c_double), C.byref(calls))
        if st:
            raise OracleError(st)
        k = it.value
        return dict(iterations=k, reason=rs.value, syndrome_ok=ok[:k], q=q[:k], posteriors=post[:k],
                    calls=calls.value)


class _OrcCfg(C.Structure):
    _fields_ = [("d_max", C.c_int32), ("use_pce", C.c_int32), ("use_vnr", C.c_int32), ("q_mode", C.c_int32),
                ("msg_clamp", C.c_double)]


class Restatement:
    """The plain-C restatement (oracle.c)."""

    def __init__(self):
        if not os.path.exists(ORC_LIB):
            raise FileNotFoundError(f"{ORC_LIB} missing (build with `make -C oracle`)")
        L = C.CDLL(ORC_LIB)
        L.orc_decode.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double),
                                 C.POINTER(C.c_uint32), C.POINTER(_OrcCfg), C.c_int, C.POINTER(C.c_uint8),
                                 C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                 C.POINTER(C.c_double)]
        L.orc_snr_for_beta.restype = C.c_double
        L.orc_snr_for_beta.argtypes = [C.c_double, C.c_double]
        L.orc_noise_normal.restype = C.c_double
        L.orc_noise_normal.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_message_bit.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_sample_frame.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_uint64, C.c_int,
                                       C.POINTER(C.c_float), C.POINTER(C.c_uint8)]
        self.L = L

    def decode(self, n_vars, check_ptr, check_vars, llr, syndrome=None, d_max=100, use_pce=True, use_vnr=False,
               q_mode=0, msg_clamp=30.0, variant=ORC_REF_DOUBLE):
        ptr = np.ascontiguousarray(check_ptr, dtype=np.int32)
        var = np.ascontiguousarray(check_vars, dtype=np.int32)
        llr = np.ascontiguousarray(llr, dtype=np.float64)
        syn = None if syndrome is None else np.ascontiguousarray(syndrome, dtype=np.uint32)
        cfg = _OrcCfg(d_max, int(use_pce), int(use_vnr), q_mode, msg_clamp)
        bits = np.zeros(n_vars, dtype=np.uint8)
        it, rs = C.c_int32(), C.c_int32()
        post = np.zeros(n_vars, dtype=np.float64)
        qt = np.full(d_max, np.nan)
        st = self.L.orc_decode(n_vars, ptr.size - 1, _p(ptr, C.c_int), _p(var, C.c_int), _p(llr, C.c_double),
                               _p(syn, C.c_uint32), C.byref(cfg), variant, _p(bits, C.c_uint8), C.byref(it),
                               C.byref(rs), _p(post, C.c_double), _p(qt, C.c_double))
        if st:
            raise OracleError(st)
        return dict(bits=bits, iterations=it.value, reason=rs.value, posteriors=post, q_trace=qt[: it.value])

    def decode_batch(self, n_vars, check_ptr, check_vars, llr, syndrome=None, **kw):
        llr = np.atleast_2d(llr)
        outs = [self.decode(n_vars, check_ptr, check_vars, llr[b], None if syndrome is None else syndrome[b], **kw)
                for b in range(llr.shape[0])]
        return dict(bits=np.stack([o["bits"] for o in outs]),
                    iterations=np.array([o["iterations"] for o in outs], dtype=np.int32),
                    reasons=np.array([o["reason"] for o in outs], dtype=np.uint8),
                    posteriors=np.stack([o["posteriors"] for o in outs]),
                    q_trace=[o["q_trace"] for o in outs])

    def snr_for_beta(self, beta, rate):
        return self.L.orc_snr_for_beta(beta, rate)

    def noise_normal(self, seed, stream, i):
        return self.L.orc_noise_normal(seed, stream, i)

    def sample_frame(self, n, snr, seed, frame, all_zero=False):
        llr = np.zeros(n, dtype=np.float32)
        x = np.zeros(n, dtype=np.uint8)
        self.L.orc_sample_frame(n, snr, seed, frame, int(all_zero), _p(llr, C.c_float), _p(x, C.c_uint8))
        return llr, x


def reference_available() -> bool:
    return os.path.exists(REF_LIB)


def restatement_available() -> bool:
    return os.path.exists(ORC_LIB)
