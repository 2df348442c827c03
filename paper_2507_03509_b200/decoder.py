"""Python mirror of the reference ``etdec`` decode interface over the C ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/core/include/etdec/*.hpp) so tests read like the
reference's own:

=======================  ====================================================
this module              reference
=======================  ====================================================
ParityCheckMatrix        etdec::ParityCheckMatrix (parity_check_matrix.hpp:12)
active_var_set           etdec::active_var_set    (parity_check_matrix.hpp:70)
load_alist/save_alist    alist.hpp:20-24
lift_protograph          protograph.hpp:31
DecodeConfig             etdec::DecodeConfig      (decoder.hpp:21-26)
StopReason               etdec::StopReason        (decoder.hpp:13-17)
DecodeOutcome            etdec::DecodeOutcome     (decoder.hpp:28-36)
BpDecoder.decode         BpDecoder::decode        (decoder.hpp:64-65)
decode                   etdec::decode            (decoder.hpp:78-79)
syndrome_check           decoder.hpp:39
vnr_statistic            decoder.hpp:42
vnr_should_stop          decoder.hpp:45
snr_for_beta             channel.hpp:24
ConfigError/IoError/     errors.hpp:8-24
ValidationError
=======================  ====================================================

``BatchDecoder.decode_batch`` is the B200-native batched entry point (many
frames per call, syndrome-aware); ``BpDecoder.decode`` is the single-frame
shim with the reference's signature.  Every decode runs the CUDA kernels;
there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib

__all__ = [
    "ConfigError", "IoError", "ValidationError", "BpdecCudaError", "BpdecOomError", "MultiDecoder",
    "ParityCheckMatrix", "ActiveVarSet", "active_var_set", "load_alist", "save_alist",
    "lift_protograph", "generate_met", "generate_met_core", "DecodeConfig", "StopReason", "DecodeOutcome",
    "BatchResult", "BpDecoder", "BatchDecoder", "decode", "syndrome_check", "vnr_statistic",
    "vnr_should_stop", "snr_for_beta", "sample_frames", "sample_frames_beta", "pack_bits", "unpack_bits",
    "PunctureMask", "no_puncture", "apply_puncture", "StopRule", "TrialStats", "wilson_interval", "run_trials",
]


class BpdecError(RuntimeError):
    status = 6


class ConfigError(BpdecError):
    """≙ etdec::ConfigError (errors.hpp:9-12), CLI exit code 1."""
    status = 1


class IoError(BpdecError):
    """≙ etdec::IoError (errors.hpp:15-18), CLI exit code 2."""
    status = 2


class ValidationError(BpdecError):
    """≙ etdec::ValidationError (errors.hpp:21-24), CLI exit code 3."""
    status = 3


class BpdecCudaError(BpdecError):
    status = 4


class BpdecOomError(BpdecError):
    status = 5


_ERRORS = {1: ConfigError, 2: IoError, 3: ValidationError, 4: BpdecCudaError, 5: BpdecOomError}


def _check(status: int) -> None:
    if status != 0:
        msg = _lib.load().bpdec_last_error().decode(errors="replace")
        raise _ERRORS.get(status, BpdecError)(msg)


def _ptr(a, ctype=None):
    """Raw address of a numpy array, a torch tensor (data_ptr) or None."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValidationError("array must be C-contiguous")
        return a.ctypes.data_as(ctype) if ctype is not None else C.c_void_p(a.ctypes.data)
    raise TypeError(f"unsupported buffer type {type(a)!r}")


# --------------------------------------------------------------------- code --
class ParityCheckMatrix:
    """Immutable Tanner graph (≙ etdec::ParityCheckMatrix).  Construct with the
    factories; ``n_vars``, ``n_checks``, ``n_edges``, ``rate()``,
    ``check_vars(c)``, ``var_degree(v)`` mirror the reference accessors."""

    def __init__(self, handle: C.c_void_p):
        self._lib = _lib.load()
        self._h = handle
        n, m, e, a = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int32()
        _check(self._lib.bpdec_code_dims(handle, C.byref(n), C.byref(m), C.byref(e), C.byref(a)))
        self.n_vars, self.n_checks, self.n_edges, self.n_active = n.value, m.value, e.value, a.value
        self._csr = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.bpdec_code_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    # ≙ from_check_lists (parity_check_matrix.cpp:10-62)
    @classmethod
    def from_check_lists(cls, n_vars: int, per_check_vars: Sequence[Sequence[int]]) -> "ParityCheckMatrix":
        ptr = np.zeros(len(per_check_vars) + 1, dtype=np.int32)
        for c, lst in enumerate(per_check_vars):
            ptr[c + 1] = ptr[c] + len(lst)
        flat = np.fromiter((v for lst in per_check_vars for v in lst), dtype=np.int64, count=int(ptr[-1]))
        if flat.size and (flat.min() < -2**31 or flat.max() >= 2**31):
            raise ValidationError("parity-check matrix: variable index out of range")
        return cls.from_csr(n_vars, len(per_check_vars), ptr, flat.astype(np.int32))

    @classmethod
    def from_csr(cls, n_vars: int, n_checks: int, check_ptr, check_vars) -> "ParityCheckMatrix":
        lib = _lib.load()
        ptr = np.ascontiguousarray(check_ptr, dtype=np.int32)
        var = np.ascontiguousarray(check_vars, dtype=np.int32)
        if ptr.size != n_checks + 1:
            raise ValidationError("parity-check matrix: check_ptr must have n_checks+1 entries")
        if ptr.size and var.size < int(ptr[-1]):
            raise ValidationError("parity-check matrix: check_vars shorter than check_ptr[-1]")
        h = C.c_void_p()
        _check(lib.bpdec_code_from_csr(n_vars, n_checks, _ptr(ptr, _lib.c_i32p), _ptr(var, _lib.c_i32p), C.byref(h)))
        return cls(h)

    def csr(self):
        if self._csr is None:
            ptr = np.zeros(self.n_checks + 1, dtype=np.int32)
            var = np.zeros(max(self.n_edges, 1), dtype=np.int32)
            _check(self._lib.bpdec_code_csr(self._h, _ptr(ptr, _lib.c_i32p), _ptr(var, _lib.c_i32p)))
            self._csr = (ptr, var[: self.n_edges])
        return self._csr

    def rate(self) -> float:
        return (self.n_vars - self.n_checks) / self.n_vars

    def check_degree(self, c: int) -> int:
        ptr, _ = self.csr()
        return int(ptr[c + 1] - ptr[c])

    def check_vars(self, c: int) -> np.ndarray:
        ptr, var = self.csr()
        return var[ptr[c]: ptr[c + 1]]

    def var_degrees(self) -> np.ndarray:
        _, var = self.csr()
        return np.bincount(var, minlength=self.n_vars).astype(np.int32)

    def var_degree(self, v: int) -> int:
        return int(self.var_degrees()[v])

    def check_degrees(self) -> np.ndarray:
        ptr, _ = self.csr()
        return np.diff(ptr).astype(np.int32)

    def syndrome(self, bits: np.ndarray) -> np.ndarray:
        """s = H x for one ([N]) or many ([F, N]) u8 words -> packed u32 words."""
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        frames = 1 if b.ndim == 1 else b.shape[0]
        out = np.zeros((frames, (self.n_checks + 31) // 32), dtype=np.uint32)
        _check(self._lib.bpdec_code_syndrome(self._h, frames, _ptr(b, _lib.c_u8p), _ptr(out, _lib.c_u32p)))
        return out[0] if b.ndim == 1 else out


@dataclass
class ActiveVarSet:
    """≙ etdec::ActiveVarSet: variables of degree >= 2, ascending."""
    members: np.ndarray


def active_var_set(code: ParityCheckMatrix) -> ActiveVarSet:
    out = np.zeros(max(code.n_active, 1), dtype=np.int32)
    _check(code._lib.bpdec_code_active_vars(code.handle, _ptr(out, _lib.c_i32p)))
    return ActiveVarSet(out[: code.n_active])


def load_alist(path: str) -> ParityCheckMatrix:
    lib = _lib.load()
    h = C.c_void_p()
    _check(lib.bpdec_code_load_alist(path.encode(), C.byref(h)))
    return ParityCheckMatrix(h)


def save_alist(code: ParityCheckMatrix, path: str) -> None:
    _check(code._lib.bpdec_code_save_alist(code.handle, path.encode()))


def lift_protograph(base: Sequence[Sequence[int]], z: int, seed: int) -> ParityCheckMatrix:
    lib = _lib.load()
    b = np.ascontiguousarray(base, dtype=np.int32)
    if b.ndim != 2:
        raise ValidationError("protograph lift: ragged base matrix")
    h = C.c_void_p()
    _check(lib.bpdec_code_lift_protograph(_ptr(b, _lib.c_i32p), b.shape[0], b.shape[1], z, seed, C.byref(h)))
    return ParityCheckMatrix(h)


def generate_met(n_vars: int, n_checks: int, frac_deg1: float, degrees: Sequence[int],
                 probs: Sequence[float], seed: int) -> ParityCheckMatrix:
    """BASELINE.json code construction (rule in csrc/code.cpp)."""
    lib = _lib.load()
    d = np.ascontiguousarray(degrees, dtype=np.int32)
    p = np.ascontiguousarray(probs, dtype=np.float64)
    if d.size != p.size:
        raise ValidationError("met generator: degree and probability lists must be aligned")
    h = C.c_void_p()
    _check(lib.bpdec_code_generate_met(n_vars, n_checks, float(frac_deg1), d.size, _ptr(d, _lib.c_i32p),
                                       _ptr(p, _lib.c_f64p), seed, C.byref(h)))
    return ParityCheckMatrix(h)


def generate_met_core(n_vars: int, n_checks: int, n_deg1: int, core_degrees: Sequence[int],
                      core_probs: Sequence[float], ext_degree: int, seed: int) -> ParityCheckMatrix:
    """Two-edge-type low-rate construction with a core code (rule in
    csrc/code.cpp, bpdec_code_generate_met_core): a code family whose FER
    falls below 1 (the BASELINE construction's never does)."""
    lib = _lib.load()
    d = np.ascontiguousarray(core_degrees, dtype=np.int32)
    p = np.ascontiguousarray(core_probs, dtype=np.float64)
    if d.size != p.size:
        raise ValidationError("met core generator: degree and probability lists must be aligned")
    h = C.c_void_p()
    _check(lib.bpdec_code_generate_met_core(int(n_vars), int(n_checks), int(n_deg1), d.size, _ptr(d, _lib.c_i32p),
                                            _ptr(p, _lib.c_f64p), int(ext_degree), seed, C.byref(h)))
    return ParityCheckMatrix(h)


# ------------------------------------------------------------------ decoder --
class StopReason(enum.IntEnum):
    """≙ etdec::StopReason (decoder.hpp:13-17)."""
    kSyndromeSatisfied = 0
    kVnrDrop = 1
    kMaxIterations = 2

    def __str__(self) -> str:  # ≙ to_string (decoder.cpp:10-17)
        return _lib.load().bpdec_stop_reason_name(int(self)).decode()


Q_RAW, Q_ABS = 0, 1


@dataclass
class DecodeConfig:
    """≙ etdec::DecodeConfig (decoder.hpp:21-26) + q-mode (RAW = reference)."""
    d_max: int = 100
    use_pce: bool = True
    use_vnr: bool = False
    msg_clamp: float = 30.0
    q_mode: int = Q_RAW

    def c_struct(self) -> _lib.Config:
        return _lib.Config(int(self.d_max), int(bool(self.use_pce)), int(bool(self.use_vnr)),
                           int(self.q_mode), float(self.msg_clamp))


@dataclass
class DecodeOutcome:
    """≙ etdec::DecodeOutcome (decoder.hpp:28-36)."""
    bits: np.ndarray
    iterations: int
    reason: StopReason
    q_trace: np.ndarray = field(default_factory=lambda: np.zeros(0))
    posteriors: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.float32))

    def converged(self) -> bool:
        return self.reason == StopReason.kSyndromeSatisfied


@dataclass
class BatchResult:
    iterations: np.ndarray
    reasons: np.ndarray
    bits: Optional[np.ndarray] = None
    posteriors: Optional[np.ndarray] = None
    q_trace: Optional[np.ndarray] = None
    syndrome_trace: Optional[np.ndarray] = None
    posterior_trace: Optional[np.ndarray] = None

    def outcome(self, f: int) -> DecodeOutcome:
        k = int(self.iterations[f])
        return DecodeOutcome(
            bits=None if self.bits is None else self.bits[f],
            iterations=k,
            reason=StopReason(int(self.reasons[f])),
            q_trace=np.zeros(0) if self.q_trace is None else self.q_trace[f, :k].copy(),
            posteriors=np.zeros(0, dtype=np.float32) if self.posteriors is None else self.posteriors[f],
        )


class BatchDecoder:
    """B200 batched decoder: a device replica of ``code`` and message state for
    ``max_slots`` frames in flight (≙ BpDecoder construction, decoder.cpp:38-48,
    once per GPU instead of once per worker thread)."""

    def __init__(self, code: ParityCheckMatrix, device: int = 0, max_slots: int = 64):
        self._lib = _lib.load()
        self.code = code
        h = C.c_void_p()
        _check(self._lib.bpdec_decoder_create(code.handle, device, max_slots, C.byref(h)))
        self._h = h
        s = C.c_int32()
        _check(self._lib.bpdec_decoder_slots(h, C.byref(s)))
        self.slots = s.value
        self.device = device

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.bpdec_decoder_destroy(h)
            self._h = None

    def __del__(self):
        self.close()

    @property
    def handle(self):
        return self._h

    def device_bytes(self) -> int:
        b = C.c_int64()
        _check(self._lib.bpdec_decoder_device_bytes(self._h, C.byref(b)))
        return b.value

    def decode_batch(self, llr, cfg: DecodeConfig, syndrome=None, *, want_bits: bool = True,
                     packed: bool = False, want_posteriors: bool = False, want_q_trace: bool = False,
                     want_syndrome_trace: bool = False, want_posterior_trace: bool = False,
                     stream: int = 0, out=None) -> BatchResult:
        """Decode ``llr`` [B, N] (float32 numpy array or torch tensor, host or
        on this decoder's device; 1-D = one frame) against ``syndrome``
        [B, ceil(M/32)] 32-bit words (None = all-zero).  Outputs are numpy
        arrays unless ``out`` (dict of preallocated buffers, validated) is
        given.  want_syndrome_trace / want_posterior_trace add the observer
        traces of bpdec_decode_batch_traced."""
        n = self.code.n_vars
        mw = (self.code.n_checks + 31) // 32
        llr = self._check_input(llr, "llr", n, (np.float32,), ("float32",))
        batch = int(llr.shape[0])
        if syndrome is not None:
            if not hasattr(syndrome, "data_ptr"):
                syndrome = np.asarray(syndrome)
                if syndrome.dtype not in (np.uint32, np.int32):
                    raise ValidationError(f"decode: syndrome must be packed 32-bit words, got {syndrome.dtype}")
                syndrome = np.ascontiguousarray(syndrome.view(np.uint32) if syndrome.dtype == np.int32 else syndrome)
            syndrome = self._check_input(syndrome, "syndrome", mw, (np.uint32, np.int32),
                                         ("int32", "uint32"), batch=batch)
        if out is None:
            out = {}
            out["iterations"] = np.zeros(batch, dtype=np.int32)
            out["reasons"] = np.zeros(batch, dtype=np.uint8)
            if want_bits:
                out["bits"] = (np.zeros((batch, (n + 31) // 32), dtype=np.uint32) if packed
                               else np.zeros((batch, n), dtype=np.uint8))
            if want_posteriors:
                out["posteriors"] = np.zeros((batch, n), dtype=np.float32)
            if want_q_trace:
                out["q_trace"] = np.zeros((batch, cfg.d_max), dtype=np.float64)
        else:
            out = dict(out)
        if want_syndrome_trace and out.get("syndrome_trace") is None:
            out["syndrome_trace"] = np.zeros((batch, cfg.d_max), dtype=np.uint8)
        if want_posterior_trace and out.get("posterior_trace") is None:
            out["posterior_trace"] = np.zeros((batch, cfg.d_max, n), dtype=np.float32)
        self._check_outputs(out, batch, n, cfg.d_max, packed)
        c = cfg.c_struct()
        flags = 1 if packed else 0
        st = C.c_void_p(stream) if stream else None
        if out.get("syndrome_trace") is not None or out.get("posterior_trace") is not None:
            _check(self._lib.bpdec_decode_batch_traced(
                self._h, batch, _ptr(llr), _ptr(syndrome), C.byref(c), flags, _ptr(out.get("bits")),
                _ptr(out["iterations"]), _ptr(out["reasons"]), _ptr(out.get("posteriors")),
                _ptr(out.get("q_trace")), _ptr(out.get("syndrome_trace")), _ptr(out.get("posterior_trace")), st))
        else:
            _check(self._lib.bpdec_decode_batch(
                self._h, batch, _ptr(llr), _ptr(syndrome), C.byref(c), flags, _ptr(out.get("bits")),
                _ptr(out["iterations"]), _ptr(out["reasons"]), _ptr(out.get("posteriors")),
                _ptr(out.get("q_trace")), st))
        return BatchResult(out["iterations"], out["reasons"], out.get("bits"), out.get("posteriors"),
                           out.get("q_trace"), out.get("syndrome_trace"), out.get("posterior_trace"))

    def _check_input(self, a, name, width, np_dtypes, torch_dtypes, batch=None):
        """Shape [B, width] (1-D = one row), dtype, contiguity and device of a
        decode input; returns the (possibly reshaped) buffer."""
        if hasattr(a, "data_ptr"):  # torch tensor
            if str(a.dtype).replace("torch.", "") not in torch_dtypes:
                raise ValidationError(f"decode: {name} tensor must be {'/'.join(torch_dtypes)}, got {a.dtype}")
            if a.dim() == 1:
                a = a.unsqueeze(0)
            if a.dim() != 2:
                raise ValidationError(f"decode: {name} must be 1-D or 2-D, got shape {tuple(a.shape)}")
            if not a.is_contiguous():
                raise ValidationError(f"decode: {name} tensor must be contiguous")
            if a.is_cuda and a.device.index != self.device:
                raise ValidationError(f"decode: {name} is on cuda:{a.device.index}, the decoder on cuda:{self.device}")
        elif isinstance(a, np.ndarray):
            if a.dtype not in np_dtypes:
                a = np.ascontiguousarray(a, dtype=np_dtypes[0])
            a = np.ascontiguousarray(a)
            if a.ndim == 1:
                a = a[None, :]
            if a.ndim != 2:
                raise ValidationError(f"decode: {name} must be 1-D or 2-D, got shape {a.shape}")
        else:
            a = np.ascontiguousarray(np.asarray(a, dtype=np_dtypes[0]))
            if a.ndim == 1:
                a = a[None, :]
        if int(a.shape[1]) != width:
            what = "does not match n_vars" if name == "llr" else "words per frame, expected"
            raise ValidationError(f"decode: {name} length {int(a.shape[1])} {what}={width}" if name == "llr" else
                                  f"decode: {name} has {int(a.shape[1])} {what} ceil(M/32)={width}")
        if batch is not None and int(a.shape[0]) != batch:
            raise ValidationError(f"decode: {name} has {int(a.shape[0])} frames, llr has {batch}")
        return a

    def _check_outputs(self, out, batch, n, d_max, packed):
        """dtype / element size / shape of the output buffers (numpy or torch)."""
        nw = (n + 31) // 32
        want = {"iterations": ((batch,), 4), "reasons": ((batch,), 1),
                "bits": (((batch, nw), 4) if packed else ((batch, n), 1)),
                "posteriors": ((batch, n), 4), "q_trace": ((batch, d_max), 8),
                "syndrome_trace": ((batch, d_max), 1), "posterior_trace": ((batch, d_max, n), 4)}
        for k in ("iterations", "reasons"):
            if out.get(k) is None:
                raise ValidationError(f"decode: output '{k}' is required")
        for k, buf in out.items():
            if buf is None:
                continue
            if k not in want:
                raise ValidationError(f"decode: unknown output '{k}'")
            shape, size = want[k]
            if hasattr(buf, "data_ptr"):
                got_shape, got_size, contig = tuple(buf.shape), buf.element_size(), buf.is_contiguous()
                if buf.is_cuda and buf.device.index != self.device:
                    raise ValidationError(f"decode: output '{k}' is on cuda:{buf.device.index}")
                fl = k in ("posteriors", "posterior_trace") and not buf.is_floating_point()
            else:
                got_shape, got_size, contig = tuple(buf.shape), buf.dtype.itemsize, buf.flags["C_CONTIGUOUS"]
                fl = k in ("posteriors", "posterior_trace") and buf.dtype.kind != "f"
            if got_shape != shape or got_size != size or not contig or fl:
                raise ValidationError(f"decode: output '{k}' must be a contiguous {shape} buffer of "
                                      f"{size}-byte elements, got {got_shape} x {got_size} B")

    def stage_inputs(self, llr, syndrome=None):
        """Starts the H2D copy of a host batch (pinned torch tensors for full
        overlap) on the decoder's copy stream; a later decode_batch with the
        same host buffers decodes from the staged copy
        (bpdec_decoder_stage_inputs)."""
        for arr, dt in ((llr, np.float32), (syndrome, np.uint32)):
            if isinstance(arr, np.ndarray) and (arr.dtype != dt or not arr.flags["C_CONTIGUOUS"]):
                raise ValidationError(f"stage_inputs: numpy inputs must be C-contiguous {np.dtype(dt).name} "
                                      "(decode_batch would otherwise copy them)")
        batch = int(llr.shape[0]) if llr.ndim > 1 else 1
        _check(self._lib.bpdec_decoder_stage_inputs(self._h, batch, _ptr(llr), _ptr(syndrome)))

    def sample_frames_device(self, snr: float, seed: int, first_frame: int, n_frames: int, llr_dev,
                             syndrome_dev=None, x_packed_dev=None, all_zero: bool = False, stream: int = 0,
                             beta_range=None):
        """Device-resident frames; beta_range=(lo, hi) draws beta_f per frame
        (config 5) and ignores `snr`."""
        st = C.c_void_p(stream) if stream else None
        if beta_range is not None:
            _check(self._lib.bpdec_decoder_sample_frames_beta_device(
                self._h, float(beta_range[0]), float(beta_range[1]), seed, first_frame, n_frames, int(all_zero),
                _ptr(llr_dev), _ptr(syndrome_dev), _ptr(x_packed_dev), st))
            return
        _check(self._lib.bpdec_decoder_sample_frames_device(
            self._h, float(snr), seed, first_frame, n_frames, int(all_zero), _ptr(llr_dev), _ptr(syndrome_dev),
            _ptr(x_packed_dev), st))

    # ------------------------------------------------------- stream mode --
    def stream_open(self, cfg: DecodeConfig, *, packed: bool = False, want_bits: bool = True,
                    want_posteriors: bool = False, want_q_trace: bool = False, ring_frames: int = 0):
        """Opens stream mode (bpdec_stream_open): batches submitted back to
        back decode as one continuous frame stream through the slots."""
        self._stream_cfg = (cfg, packed, want_bits, want_posteriors, want_q_trace)
        c = cfg.c_struct()
        _check(self._lib.bpdec_stream_open(self._h, C.byref(c), 1 if packed else 0, int(ring_frames),
                                           int(want_bits), int(want_posteriors), int(want_q_trace)))
        self._stream_keep = {}

    def stream_submit(self, llr, syndrome=None, out=None) -> int:
        """Submits a batch; returns its ticket.  ``out`` (dict of buffers:
        iterations, reasons, bits, posteriors, q_trace — host arrays/tensors,
        pinned for overlap, or device tensors) receives the outputs when the
        batch completes (stream_wait).  Inputs must stay untouched until then."""
        cfg, packed, want_bits, want_post, want_q = self._stream_cfg
        n = self.code.n_vars
        mw = (self.code.n_checks + 31) // 32
        llr = self._check_input(llr, "llr", n, (np.float32,), ("float32",))
        batch = int(llr.shape[0])
        if syndrome is not None:
            syndrome = self._check_input(syndrome, "syndrome", mw, (np.uint32, np.int32), ("int32", "uint32"),
                                         batch=batch)
        if out is None:
            out = {"iterations": np.zeros(batch, dtype=np.int32), "reasons": np.zeros(batch, dtype=np.uint8)}
            if want_bits:
                out["bits"] = (np.zeros((batch, (n + 31) // 32), dtype=np.uint32) if packed
                               else np.zeros((batch, n), dtype=np.uint8))
            if want_post:
                out["posteriors"] = np.zeros((batch, n), dtype=np.float32)
            if want_q:
                out["q_trace"] = np.zeros((batch, cfg.d_max), dtype=np.float64)
        self._check_outputs(out, batch, n, cfg.d_max, packed)
        t = C.c_int64()
        _check(self._lib.bpdec_stream_submit(
            self._h, batch, _ptr(llr), _ptr(syndrome), _ptr(out.get("bits")), _ptr(out["iterations"]),
            _ptr(out["reasons"]), _ptr(out.get("posteriors")), _ptr(out.get("q_trace")), C.byref(t)))
        self._stream_keep[t.value] = (llr, syndrome, out)  # alive until waited for
        return t.value

    def stream_wait(self, ticket: int) -> BatchResult:
        try:
            _check(self._lib.bpdec_stream_wait(self._h, int(ticket)))
        finally:
            keep = self._stream_keep.pop(int(ticket), None)
        out = keep[2] if keep else {}
        return BatchResult(out.get("iterations"), out.get("reasons"), out.get("bits"), out.get("posteriors"),
                           out.get("q_trace"))

    def stream_query(self, ticket: int) -> bool:
        d = C.c_int32()
        _check(self._lib.bpdec_stream_query(self._h, int(ticket), C.byref(d)))
        return bool(d.value)

    def stream_timer_reset(self):
        """Arms the stream's device timer (no batch may be in flight)."""
        _check(self._lib.bpdec_stream_timer_reset(self._h))

    def stream_device_ms(self) -> float:
        """CUDA-event time from the first step launched after
        stream_timer_reset to the last completed batch's output copy."""
        ms = C.c_double()
        _check(self._lib.bpdec_stream_device_ms(self._h, C.byref(ms)))
        return ms.value

    def stream_close(self):
        try:
            _check(self._lib.bpdec_stream_close(self._h))
        finally:
            self._stream_keep = {}

    # profiling (CUDA events on the launching stream)
    KERNELS = ("check", "variable", "decide", "turnover", "compact")
    _KERNEL_IDS = {"check": 0, "variable": 1, "decide": 2, "turnover": 4, "compact": 5}

    def set_profiling(self, enable: bool):
        _check(self._lib.bpdec_decoder_set_profiling(self._h, int(enable)))

    def reset_profile(self):
        _check(self._lib.bpdec_decoder_reset_profile(self._h))

    def profile(self) -> dict:
        res = {}
        for name in self.KERNELS:
            ms, n, fi = C.c_double(), C.c_int64(), C.c_double()
            _check(self._lib.bpdec_decoder_profile(self._h, self._KERNEL_IDS[name], C.byref(ms), C.byref(n),
                                                   C.byref(fi)))
            res[name] = {"ms": ms.value, "launches": n.value}
            res["frame_iterations"] = fi.value
        return res

    def launch_count(self) -> int:
        n = C.c_int64()
        _check(self._lib.bpdec_decoder_launch_count(self._h, C.byref(n)))
        return n.value


class MultiDecoder:
    """Frame-sharded decoding over several GPUs of one host
    (bpdec_multi_*): one decoder per entry of ``devices`` (a
    device may repeat), a host thread each, frames dealt from a shared chunk
    queue, outputs gathered into the caller's buffers at their frame index."""

    def __init__(self, code: ParityCheckMatrix, devices: Sequence[int], slots_per_decoder: int = 64):
        self._lib = _lib.load()
        self.code = code
        dv = np.ascontiguousarray(list(devices), dtype=np.int32)
        h = C.c_void_p()
        _check(self._lib.bpdec_multi_create(code.handle, _ptr(dv, _lib.c_i32p), int(dv.size), int(slots_per_decoder),
                                            C.byref(h)))
        self._h = h
        self.devices = list(devices)
        self.last_frames_per_decoder = None

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.bpdec_multi_destroy(h)
            self._h = None

    def __del__(self):
        self.close()

    def decode_batch(self, llr, cfg: DecodeConfig, syndrome=None, *, want_bits: bool = True, packed: bool = False,
                     want_posteriors: bool = False, want_q_trace: bool = False, chunk_frames: int = 0,
                     out=None) -> BatchResult:
        n = self.code.n_vars
        mw = (self.code.n_checks + 31) // 32
        llr = np.ascontiguousarray(llr, dtype=np.float32) if not hasattr(llr, "data_ptr") else llr
        if llr.ndim == 1:
            llr = llr[None, :]
        if llr.shape[1] != n:
            raise ValidationError(f"decode: LLR length {llr.shape[1]} does not match n_vars={n}")
        batch = int(llr.shape[0])
        if syndrome is not None and not hasattr(syndrome, "data_ptr"):
            syndrome = np.ascontiguousarray(syndrome).view(np.uint32).reshape(batch, -1)
            if syndrome.shape[1] != mw:
                raise ValidationError(f"decode: syndrome has {syndrome.shape[1]} words per frame, expected {mw}")
        if out is None:
            out = {"iterations": np.zeros(batch, dtype=np.int32), "reasons": np.zeros(batch, dtype=np.uint8)}
            if want_bits:
                out["bits"] = (np.zeros((batch, (n + 31) // 32), dtype=np.uint32) if packed
                               else np.zeros((batch, n), dtype=np.uint8))
            if want_posteriors:
                out["posteriors"] = np.zeros((batch, n), dtype=np.float32)
            if want_q_trace:
                out["q_trace"] = np.zeros((batch, cfg.d_max), dtype=np.float64)
        taken = np.zeros(len(self.devices), dtype=np.int64)
        c = cfg.c_struct()
        _check(self._lib.bpdec_multi_decode_batch(
            self._h, batch, _ptr(llr), _ptr(syndrome), C.byref(c), 1 if packed else 0, _ptr(out.get("bits")),
            _ptr(out["iterations"]), _ptr(out["reasons"]), _ptr(out.get("posteriors")), _ptr(out.get("q_trace")),
            int(chunk_frames), _ptr(taken, _lib.c_i64p)))
        self.last_frames_per_decoder = taken
        return BatchResult(out["iterations"], out["reasons"], out.get("bits"), out.get("posteriors"),
                           out.get("q_trace"))


class BpDecoder:
    """Single-frame shim with the reference signature (decoder.hpp:57-65):
    ``BpDecoder(code).decode(llr_in, active, cfg, observer)`` -> DecodeOutcome.
    LLRs are rounded to float32 (the decoder's input type).

    ``active`` must be ``active_var_set(code)`` (or None): the device q
    statistic is built over the degree>=2 variables; another set raises
    ValidationError instead of being silently ignored.  ``observer(iteration,
    posteriors, syndrome_ok, q)`` is replayed after the decode from the
    per-iteration traces (bpdec_decode_batch_traced) with the same arguments
    the reference passes (decoder.cpp:107-112): syndrome_ok is computed every
    iteration, PCE on or off, and posteriors are that iteration's (float32
    values as float64)."""

    def __init__(self, code: ParityCheckMatrix, device: int = 0):
        self.code = code
        self._dec = BatchDecoder(code, device=device, max_slots=32)
        self._active = None

    def _check_active(self, active: Optional[ActiveVarSet]):
        if active is None:
            return
        if self._active is None:
            self._active = active_var_set(self.code).members
        m = np.asarray(active.members, dtype=np.int64)
        if m.shape != self._active.shape or not np.array_equal(m, self._active):
            raise ValidationError("decode: only active_var_set(code) (the degree>=2 variables) is supported as the "
                                  "VNR active set")

    def decode(self, llr_in, active: Optional[ActiveVarSet] = None, cfg: Optional[DecodeConfig] = None,
               syndrome=None, observer=None) -> DecodeOutcome:
        cfg = cfg or DecodeConfig()
        llr = np.asarray(llr_in, dtype=np.float64)
        if llr.ndim != 1 or llr.size != self.code.n_vars:
            raise ValidationError(f"decode: LLR length {llr.size} does not match n_vars={self.code.n_vars}")
        if not np.all(np.isfinite(llr)):
            raise ValidationError("decode: non-finite input LLR")
        self._check_active(active)
        l32 = llr.astype(np.float32)[None, :]
        syn = None if syndrome is None else np.asarray(syndrome, dtype=np.uint32)[None, :]
        r = self._dec.decode_batch(l32, cfg, syn, want_posteriors=True, want_q_trace=True,
                                   want_syndrome_trace=observer is not None)
        out = r.outcome(0)
        if observer is not None:
            k = out.iterations
            # per-iteration posteriors: the decode is deterministic per frame,
            # so a second run with d_max = k traces exactly the iterations the
            # first one ran (bounded trace buffer: k x N floats)
            tcfg = DecodeConfig(d_max=k, use_pce=False, use_vnr=False, msg_clamp=cfg.msg_clamp, q_mode=cfg.q_mode)
            t = self._dec.decode_batch(l32, tcfg, syn, want_bits=False, want_posterior_trace=True)
            for it in range(k):
                observer(it + 1, t.posterior_trace[0, it].astype(np.float64), bool(r.syndrome_trace[0, it] == 1),
                         float(out.q_trace[it]))
        return out


def decode(code: ParityCheckMatrix, llr_in, active: Optional[ActiveVarSet], cfg: DecodeConfig,
           syndrome=None) -> DecodeOutcome:
    """≙ etdec::decode (decoder.hpp:78-79): throwaway decoder."""
    return BpDecoder(code).decode(llr_in, active, cfg, syndrome=syndrome)


def syndrome_check(code: ParityCheckMatrix, bits, syndrome=None) -> bool:
    """≙ syndrome_check (decoder.cpp:19-30); optional target syndrome."""
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    if b.size != code.n_vars:
        raise ValidationError(
            f"syndrome_check: bit vector length {b.size} does not match n_vars={code.n_vars}")
    s = None if syndrome is None else np.ascontiguousarray(syndrome, dtype=np.uint32)
    ok = C.c_int32()
    _check(code._lib.bpdec_syndrome_check(code.handle, _ptr(b, _lib.c_u8p), _ptr(s, _lib.c_u32p), C.byref(ok)))
    return bool(ok.value)


def vnr_statistic(posteriors, active: ActiveVarSet) -> float:
    """≙ vnr_statistic (decoder.cpp:32-36): sequential double sum."""
    q = 0.0
    p = np.asarray(posteriors, dtype=np.float64)
    for v in active.members:
        q += float(p[v])
    return q


def vnr_should_stop(q_k: float, q_km1: float) -> bool:
    """≙ vnr_should_stop (decoder.hpp:45): strict decrease."""
    return q_k < q_km1


def snr_for_beta(beta: float, rate: float) -> float:
    """≙ snr_for_beta (channel.cpp:29-42): snr = 2^(2R/beta) - 1."""
    out = C.c_double()
    _check(_lib.load().bpdec_snr_for_beta(float(beta), float(rate), C.byref(out)))
    return out.value


def sample_frames(code: ParityCheckMatrix, snr: float, seed: int, first_frame: int, n_frames: int,
                  all_zero: bool = False):
    """Seeded syndrome-mode frames -> (llr [F,N] f32, x [F,N] u8, s [F,MW] u32)."""
    llr = np.zeros((n_frames, code.n_vars), dtype=np.float32)
    x = np.zeros((n_frames, code.n_vars), dtype=np.uint8)
    s = np.zeros((n_frames, (code.n_checks + 31) // 32), dtype=np.uint32)
    _check(code._lib.bpdec_sample_frames(code.handle, float(snr), seed, first_frame, n_frames, int(all_zero),
                                         _ptr(llr, _lib.c_f32p), _ptr(x, _lib.c_u8p), _ptr(s, _lib.c_u32p)))
    return llr, x, s


def sample_frames_beta(code: ParityCheckMatrix, beta_lo: float, beta_hi: float, seed: int, first_frame: int,
                       n_frames: int, all_zero: bool = False):
    """Mixed-SNR frames (config 5): beta_f ~ U[lo, hi] per frame ->
    (llr, x, s, snr[F])."""
    llr = np.zeros((n_frames, code.n_vars), dtype=np.float32)
    x = np.zeros((n_frames, code.n_vars), dtype=np.uint8)
    s = np.zeros((n_frames, (code.n_checks + 31) // 32), dtype=np.uint32)
    snr = np.zeros(n_frames, dtype=np.float64)
    _check(code._lib.bpdec_sample_frames_beta(code.handle, float(beta_lo), float(beta_hi), seed, first_frame, n_frames,
                                              int(all_zero), _ptr(llr, _lib.c_f32p), _ptr(x, _lib.c_u8p),
                                              _ptr(s, _lib.c_u32p), _ptr(snr, _lib.c_f64p)))
    return llr, x, s, snr


# ------------------------------------------------------- Monte-Carlo harness --
@dataclass
class PunctureMask:
    """≙ etdec::PunctureMask (puncture.hpp:14-21)."""
    punctured: np.ndarray
    effective_rate: float

    def empty(self) -> bool:
        return self.punctured.size == 0


def no_puncture(code: ParityCheckMatrix) -> PunctureMask:
    return PunctureMask(np.zeros(0, dtype=np.int32), code.rate())


def apply_puncture(code: ParityCheckMatrix, target_rate: float, seed: int) -> PunctureMask:
    """≙ apply_puncture (puncture.cpp:16-48), same positions for the same seed."""
    out = np.zeros(code.n_vars, dtype=np.int32)
    cnt = C.c_int32()
    eff = C.c_double()
    _check(code._lib.bpdec_code_apply_puncture(code.handle, float(target_rate), seed, _ptr(out, _lib.c_i32p),
                                               C.byref(cnt), C.byref(eff)))
    return PunctureMask(out[: cnt.value].copy(), eff.value)


@dataclass
class StopRule:
    """≙ etdec::StopRule (channel.hpp:42-45)."""
    min_frame_errors: int = 100
    max_frames: int = 10000


@dataclass
class TrialStats:
    """≙ etdec::TrialStats (channel.hpp:47-61)."""
    frames: int
    frame_errors: int
    undetected_errors: int
    fer: float
    fer_ci_low: float
    fer_ci_high: float
    d_bar: float
    iteration_sum: int
    iteration_histogram: dict
    stops_syndrome: int
    stops_vnr: int
    stops_max_iter: int
    hit_max_frames: bool


def wilson_interval(k: int, n: int):
    """≙ wilson_interval (channel.cpp:63-72)."""
    lo, hi = C.c_double(), C.c_double()
    _check(_lib.load().bpdec_wilson_interval(int(k), int(n), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def run_trials(dec: "BatchDecoder", snr: float, cfg: DecodeConfig, stop: StopRule, master_seed: int,
               mask: Optional[PunctureMask] = None, block: Optional[int] = None) -> TrialStats:
    """≙ run_trials (channel.cpp:74-156) on the GPU: trials 0,1,2,... of the
    all-zero codeword, prefix-exact stop rule; results do not depend on
    `block` (frames decoded per device batch, default = the decoder's slots)."""
    lib = dec._lib
    p = None if mask is None or mask.empty() else np.ascontiguousarray(mask.punctured, dtype=np.int32)
    st = _lib.TrialStatsC()
    hist = np.zeros(cfg.d_max + 1, dtype=np.int64)
    c = cfg.c_struct()
    sr = _lib.StopRule(int(stop.min_frame_errors), int(stop.max_frames))
    _check(lib.bpdec_run_trials(dec.handle, float(snr), _ptr(p, _lib.c_i32p), 0 if p is None else p.size, C.byref(c),
                                C.byref(sr), master_seed, int(block or dec.slots), C.byref(st),
                                _ptr(hist, _lib.c_i64p)))
    return TrialStats(st.frames, st.frame_errors, st.undetected_errors, st.fer, st.fer_ci_low, st.fer_ci_high,
                      st.d_bar, st.iteration_sum, {int(k): int(v) for k, v in enumerate(hist) if v},
                      st.stops_syndrome, st.stops_vnr, st.stops_max_iter, bool(st.hit_max_frames))


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """u8 [.., N] -> u32 [.., ceil(N/32)] LSB-first."""
    b = np.asarray(bits, dtype=np.uint8)
    n = b.shape[-1]
    pad = (-n) % 32
    if pad:
        b = np.concatenate([b, np.zeros(b.shape[:-1] + (pad,), dtype=np.uint8)], axis=-1)
    return np.packbits(b.reshape(b.shape[:-1] + (-1, 32)), axis=-1, bitorder="little").view(np.uint32)[..., 0]


def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    w = np.ascontiguousarray(words, dtype=np.uint32)
    b = np.unpackbits(w.view(np.uint8), bitorder="little")
    return b.reshape(w.shape[:-1] + (-1,))[..., :n]
