#!/usr/bin/env python3
"""Benchmark of the batched VNR-ET / PCE-ET LDPC decode hot path.

Our arm (default):   python bench.py [--gpus N --steps K --warmup W]
Reference arm:       python bench.py --impl reference [...]

A step = one decode of one batch of BASELINE configs[1] (cfg2: R=0.1,
N=2^20, 64 frames per GPU, D_max=500, beta=0.95, syndrome mode, VNR-ET with
PCE) with inputs resident in HBM.  Multi-GPU: one process per GPU (torchrun),
frames sharded by global frame index, no collective on the decode path
("scaling": "weak"); the timed region is bracketed by barrier + synchronize
and the max over ranks is reported.

Metric: edge-updates/s = sum_f iterations_f * E / time, plus
decoded / processed info bits/s and the mean iterations of VNR vs PCE.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edge_updates_per_s"
UNIT = "edge-updates/s"
E_BYTES_MODEL_A = None  # filled per code: 16E + 4N + (N+M)/8 per frame-iteration


# frames per GPU per step for each BASELINE workload (cfg4/cfg5 are the
# 8-GPU streams 512..4096 / 8192 frames; per GPU at N=1 the first shard)
E2E_RUNS = 5  # e2e: median of this many timed runs (>= 5)

FRAMES = {"cfg1": 16, "cfg2": 64, "cfg3": 32, "cfg4": 512, "cfg5": 1024, "met": 64, "met_s": 16}


def workload_beta(args):
    """(beta, beta_range) for the workload: fixed beta, or a per-frame range."""
    if args.workload == "cfg5" and args.beta is None:
        return None, (0.92, 1.0)
    if args.beta is not None:
        return args.beta, None
    # cfg2/cfg4: the middle of configs[1]'s swept grid (0.92 .. 0.99); met:
    # inside its waterfall (FER between 0 and 1)
    return {"cfg3": 0.98, "met": 0.87, "met_s": 0.8}.get(args.workload, 0.96), None


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--beta", type=float, default=None,
                    help="reconciliation efficiency (default 0.95; cfg3 0.98; cfg5 draws U[0.92,1] per frame)")
    ap.add_argument("--frames", type=int, default=None, help="frames per GPU per step")
    ap.add_argument("--slots", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pce-compare", action="store_true")
    ap.add_argument("--cpu-frames", type=int, default=None)
    ap.add_argument("--clock-ms", type=int, default=200, help="nvidia-smi sampling period during the timed region")
    ap.add_argument("--no-clocks", action="store_true", help="diagnostics: no nvidia-smi sampling")
    ap.add_argument("--mode", choices=["stream", "batch"], default="stream",
                    help="stream: the K batches go through bpdec_stream_* back to back (a batch's tail lanes are "
                         "refilled with the next batch's frames); batch: one blocking bpdec_decode_batch per step")
    ap.add_argument("--multi", action="store_true",
                    help="strong scaling in ONE process: the K x F frames of the run split over --gpus devices "
                         "by bpdec_multi_decode_batch (dynamic chunk queue, host gather)")
    ap.add_argument("--multi-devices", default=None,
                    help="--multi: comma-separated device list (a device may repeat; default 0..gpus-1)")
    ap.add_argument("--no-traffic", action="store_true", help="skip the live ncu DRAM-traffic probe of k_check")
    ap.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--ref-inputs", default=None, help=argparse.SUPPRESS)
    return ap.parse_args()


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def spawn_ranks(args):
    """`--gpus N` without a torchrun environment: relaunch this command as N
    local ranks (one process per GPU, 127.0.0.1 rendezvous) and return the
    launcher's exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------ clocks --
def gpu_uuid(dev):
    """NVML / nvidia-smi identity of CUDA device `dev` (robust to
    CUDA_VISIBLE_DEVICES renumbering); the CUDA ordinal if unknown."""
    import torch
    try:
        u = str(torch.cuda.get_device_properties(dev).uuid)
        return u if u.startswith("GPU-") else "GPU-" + u
    except Exception:
        return dev


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML
    polled every few ms from a thread (pynvml), else `nvidia-smi -lms`."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int, period_ms: int = 200):
        self.index = index
        self.period = period_ms
        self.proc = None
        self.nvml = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reasons set) from NVML
        self.running = False

    def start(self, enabled=True):
        if not enabled:
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = (pynvml.nvmlDeviceGetHandleByUUID(self.index) if isinstance(self.index, str)
                      else pynvml.nvmlDeviceGetHandleByIndex(self.index))
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.running = True
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            while not self.samples and self.t.is_alive():
                time.sleep(0.001)
            self.samples.clear()
            return
        except Exception:  # no pynvml / NVML: fall back to nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's NVML start-up must not overlap the timed region
            t0 = time.time()
            while not self.lines and time.time() - t0 < 10:
                time.sleep(0.05)
            self.lines.clear()
        except OSError:
            self.proc = None

    def _poll(self):
        p = self.nvml
        bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}
        get_reasons = getattr(p, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            p.nvmlDeviceGetCurrentClocksThrottleReasons
        while self.running:
            try:
                sm = p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM)
                r = get_reasons(self.h)
                self.samples.append((float(sm), float(self.max_sm), {n for n, b in bits.items() if r & b}))
            except Exception:
                break
            time.sleep(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            self.running = False
            self.t.join(timeout=2)
            smp = list(self.samples)
            reasons = set().union(*[x[2] for x in smp]) if smp else set()
            return {"sm_mhz": float(np.median([x[0] for x in smp])) if smp else None,
                    "sm_max_mhz": max(x[1] for x in smp) if smp else None,
                    "reasons": sorted(reasons), "samples": len(smp), "source": "nvml"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for k, nm in enumerate(self.NAMES):
                if p[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


# -------------------------------------------------------- distributed --
def dist_setup(n_gpus):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        return rank, ws, local, dist
    return 0, 1, 0, None


def max_over_ranks(x: float, dist) -> float:
    if dist is None:
        return x
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, dist) -> float:
    if dist is None:
        return x
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def shard(total_frames: int, rank: int, world: int):
    """Contiguous shard of global frame indices for `rank`."""
    per = (total_frames + world - 1) // world
    a = min(total_frames, rank * per)
    return a, min(total_frames, a + per)


# ------------------------------------------------------------- helpers --
def model_bytes(code):
    """Model A bytes per frame-iteration and the per-kernel
    split (check pass: v2c read + c2v write = 8E)."""
    E, N, M = code.n_edges, code.n_vars, code.n_checks
    return 16 * E + 4 * N + (N + M) / 8.0, 8.0 * E


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def cpu_reference_time(code, llr_eq, d_max, threads):
    """Reference decoder (oracle/_ref) on host cores: returns (seconds,
    total iterations, reasons)."""
    import oracle
    R = oracle.Reference()
    ptr, var = code.csr()
    rc = R.code_from_csr(code.n_vars, code.n_checks, ptr, var)
    t0 = time.perf_counter()
    r = rc.decode_batch(llr_eq, d_max=d_max, use_pce=True, use_vnr=True, threads=threads,
                        want_posteriors=False, want_q_trace=False)
    dt = time.perf_counter() - t0
    return dt, int(r["iterations"].sum()), r


def emit(obj):
    print(json.dumps(obj), flush=True)


# ------------------------------------------------------ reference arm --
def write_reference_inputs(args):
    """Child process of the reference arm: generates the workload's code and
    frames (this repo's seeded generator) and writes them as .npy files, so
    the timing process maps only the reference library (oracle/_ref)."""
    import paper_2507_03509_b200 as P
    w = P.WORKLOADS[args.workload]
    code = w.make_code()
    threads = os.cpu_count() or 1
    frames = args.cpu_frames or threads
    beta, brange = workload_beta(args)
    if brange is None:
        llr, x, _ = P.sample_frames(code, P.snr_for_beta(beta, code.rate()), P.FRAME_SEED, 0, frames)
    else:
        llr, x, _, _ = P.sample_frames_beta(code, brange[0], brange[1], P.FRAME_SEED, 0, frames)
    leq = (llr * (1 - 2 * x.astype(np.float32))).astype(np.float64)
    ptr, var = code.csr()
    d = args.ref_inputs
    np.save(os.path.join(d, "check_ptr.npy"), ptr)
    np.save(os.path.join(d, "check_vars.npy"), var)
    np.save(os.path.join(d, "llr.npy"), leq)
    with open(os.path.join(d, "meta.json"), "w") as f:
        json.dump({"name": w.name, "n_vars": code.n_vars, "n_checks": code.n_checks, "d_max": w.d_max,
                   "beta": beta if brange is None else list(brange), "frames": frames}, f)


def run_reference(args):
    """Rank 0 alone times the reference CPU decoder; other ranks exit.  The
    code and frames come from files written by a child process, so this
    process loads no library of this repo: only oracle/_ref (the unmodified
    reference compiled from its sources)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    import tempfile
    import oracle
    if not oracle.reference_available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/libetdec_ref.so not built (needs /root/reference)"})
        return
    with tempfile.TemporaryDirectory() as td:
        cmd = [sys.executable, os.path.abspath(__file__), "--ref-inputs", td, "--workload", args.workload]
        for flag, v in (("--beta", args.beta), ("--cpu-frames", args.cpu_frames)):
            if v is not None:
                cmd += [flag, str(v)]
        subprocess.run(cmd, check=True, env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
        with open(os.path.join(td, "meta.json")) as f:
            meta = json.load(f)
        ptr = np.load(os.path.join(td, "check_ptr.npy"))
        var = np.load(os.path.join(td, "check_vars.npy"))
        leq = np.load(os.path.join(td, "llr.npy"))
    threads = os.cpu_count() or 1
    frames = meta["frames"]
    R = oracle.Reference()
    rc = R.code_from_csr(meta["n_vars"], meta["n_checks"], ptr, var)
    n_edges = int(var.size)
    times, iters = [], []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = rc.decode_batch(leq, d_max=meta["d_max"], use_pce=True, use_vnr=True, threads=threads,
                            want_posteriors=False, want_q_trace=False)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            times.append(dt)
            iters.append(int(r["iterations"].sum()))
    T = float(np.sum(times))
    value = float(np.sum(iters)) * n_edges / T
    sample = (f"{frames} frames of {meta['name']} (beta={meta['beta']}, VNR+PCE, D_max={meta['d_max']}) per step, "
              f"all-zero-equivalent inputs L*(1-2x), s=0 (the reference's semantics); code and frames read from "
              f"files written by a child process")
    emit({"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
          "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times),
          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
          "data": "synthetic (seeded BASELINE generator)",
          "config": {"workload": meta["name"], "frames_per_step": frames, "beta": meta["beta"],
                     "d_max": meta["d_max"], "et": "vnr+pce", "threads": threads},
          "d_bar": float(np.sum(iters)) / (frames * len(times)),
          "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                           "cpu_model": cpu_model(), "sample": sample},
          "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})


# ------------------------------------------------------------- our arm --
def layout_bytes(code):
    """Model B: the bytes THIS layout must move per
    frame-iteration.  Check pass 8(E_hi - n11) + 4 N1 (previous c2v read and
    new c2v written for edges to degree>=2 variables except the constant
    (1,1) checks, degree-1 LLRs read); variable pass 4 E_hi + 8 N_V (c2v
    gathered, LLR read, posterior written)."""
    ptr, var = code.csr()
    vdeg = np.bincount(var, minlength=code.n_vars)
    hi = vdeg[var] >= 2
    cidx = np.repeat(np.arange(code.n_checks), np.diff(ptr))
    nh = np.bincount(cidx[hi], minlength=code.n_checks)
    nd = np.bincount(cidx[vdeg[var] == 1], minlength=code.n_checks)
    e_hi, n1, n_v = int(hi.sum()), int(np.sum(vdeg == 1)), int(np.sum(vdeg >= 2))
    n11 = int(np.sum((nh == 1) & (nd == 1)))
    return {"check": 8.0 * (e_hi - n11) + 4.0 * n1, "variable": 4.0 * e_hi + 8.0 * n_v,
            "e_hi": e_hi, "n_deg1": n1, "n_v": n_v, "n11": n11}


def make_frames(P, dec, code, args, F, first, stream_ptr):
    import torch
    beta, brange = workload_beta(args)
    snr = P.snr_for_beta(beta, code.rate()) if brange is None else 0.0
    N, M = code.n_vars, code.n_checks
    MW, NW = (M + 31) // 32, (N + 31) // 32
    d_llr = torch.empty((F, N), dtype=torch.float32, device="cuda")
    d_syn = torch.empty((F, MW), dtype=torch.int32, device="cuda")
    d_x = torch.empty((F, NW), dtype=torch.int32, device="cuda")
    dec.sample_frames_device(snr, P.FRAME_SEED, first, F, d_llr, d_syn, d_x, stream=stream_ptr, beta_range=brange)
    return d_llr, d_syn, d_x


def traffic_probe(args):
    """Runs under ncu (measure_traffic): the bench's decode of one workload
    batch in the bench's mode, nothing else on the GPU; prints the
    frame-iterations and k_check launches it made."""
    import torch
    import paper_2507_03509_b200 as P
    from paper_2507_03509_b200.decoder import Q_ABS
    w = P.WORKLOADS[args.workload]
    code = w.make_code()
    F = args.frames or FRAMES[args.workload]
    dec = P.BatchDecoder(code, device=0, max_slots=args.slots or
                         (min(6 * F, 1024) if args.mode == "stream" else min(F, 512)))
    d_llr, d_syn, _ = make_frames(P, dec, code, args, F, 0, 0)
    torch.cuda.synchronize()
    cfg = P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=True, q_mode=Q_ABS)
    dec.reset_profile()
    dec.set_profiling(True)
    if args.mode == "stream":
        dec.stream_open(cfg, packed=True)
        outs = [{"iterations": torch.zeros(F, dtype=torch.int32, device="cuda"),
                 "reasons": torch.zeros(F, dtype=torch.uint8, device="cuda"),
                 "bits": torch.zeros((F, (code.n_vars + 31) // 32), dtype=torch.int32, device="cuda")}
                for _ in range(8)]  # enough batches for the stream's steady state
        for t in [dec.stream_submit(d_llr, d_syn, out=o) for o in outs]:
            dec.stream_wait(t)
        dec.stream_close()
    else:
        dec.decode_batch(d_llr, cfg, syndrome=d_syn, packed=True)
    prof = dec.profile()
    print("TRAFFIC_PROBE " + json.dumps({"frame_iterations": prof["frame_iterations"],
                                         "check_launches": prof["check"]["launches"]}), flush=True)


def measure_traffic(args, timeout_s=300):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of every
    k_check launch of one bench batch, measured now by ncu in a child
    process (traffic_probe).  Returns a dict or None with the reason."""
    import csv
    import shutil
    import tempfile
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    with tempfile.TemporaryDirectory() as td:
        log = os.path.join(td, "ncu.csv")
        cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "-k", "regex:k_check",
               "--clock-control", "none", "--print-units", "base", "--csv", "--log-file", log,
               sys.executable, os.path.abspath(__file__), "--traffic-probe", "--workload", args.workload,
               "--mode", args.mode]
        for flag, v in (("--frames", args.frames), ("--slots", args.slots), ("--beta", args.beta)):
            if v is not None:
                cmd += [flag, str(v)]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s)
        except subprocess.TimeoutExpired:
            return None, f"ncu probe timed out after {timeout_s} s"
        probe = None
        for ln in r.stdout.splitlines():
            if ln.startswith("TRAFFIC_PROBE "):
                probe = json.loads(ln[len("TRAFFIC_PROBE "):])
        if r.returncode != 0 or probe is None or not os.path.exists(log):
            return None, f"ncu probe failed (rc {r.returncode}): {(r.stderr or r.stdout)[-200:]}"
        per = {}
        with open(log) as f:
            rows = [ln for ln in f if ln.startswith('"')]
        for row in csv.DictReader(rows):
            try:
                per.setdefault(row["ID"], 0.0)
                per[row["ID"]] += float(row["Metric Value"].replace(",", ""))
            except (KeyError, ValueError):
                continue
    if not per:
        return None, "ncu probe: no k_check launches in the CSV"
    total = float(sum(per.values()))
    return {"bytes_per_launch": total / len(per), "launches": len(per), "total_bytes": total,
            "frame_iterations": probe["frame_iterations"],
            "bytes_per_frame_iteration": total / max(probe["frame_iterations"], 1.0)}, None


def run_ours(args):
    rank, world, local, dist = dist_setup(args.gpus)
    import torch
    import paper_2507_03509_b200 as P
    from paper_2507_03509_b200.decoder import Q_ABS

    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench: rank {rank} needs cuda:{local}, only {torch.cuda.device_count()} device(s) visible")
    torch.cuda.set_device(local)
    w = P.WORKLOADS[args.workload]
    code = w.make_code()
    F = args.frames or FRAMES[args.workload]
    # stream mode keeps six batches' worth of slots in flight: a batch's
    # tail shares the steps with the next batches' frames
    slots = args.slots or (min(6 * F, 1024) if args.mode == "stream" else min(F, 512))
    beta, brange = workload_beta(args)
    dec = P.BatchDecoder(code, device=local, max_slots=slots)
    # weak scaling: rank r owns global frames [r*F, (r+1)*F)
    first = rank * F
    N, M = code.n_vars, code.n_checks
    MW, NW = (M + 31) // 32, (N + 31) // 32
    stream = torch.cuda.Stream(device=local)
    sptr = stream.cuda_stream
    d_llr, d_syn, d_x = make_frames(P, dec, code, args, F, first, sptr)
    torch.cuda.synchronize()
    cfg = P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=True, q_mode=Q_ABS)
    K = max(1, args.steps)
    use_stream = args.mode == "stream"

    def dev_out():
        return {"iterations": torch.zeros(F, dtype=torch.int32, device="cuda"),
                "reasons": torch.zeros(F, dtype=torch.uint8, device="cuda"),
                "bits": torch.zeros((F, NW), dtype=torch.int32, device="cuda")}

    out = dev_out()

    def batch_step():
        return dec.decode_batch(d_llr, cfg, syndrome=d_syn, packed=True, out=out, stream=sptr)

    # stream mode: one output set per in-flight batch (a step's outputs are
    # final when its ticket completes)
    souts = [dev_out() for _ in range(K)] if use_stream else None

    def stream_run(nsteps, llr_src, syn_src, outs):
        """nsteps batches through the open stream back to back; returns the
        summed iterations (the host read of every step's result)."""
        tickets = [dec.stream_submit(llr_src(k), syn_src(k), out=outs[k % len(outs)]) for k in range(nsteps)]
        it = 0
        for k, t in enumerate(tickets):
            dec.stream_wait(t)
            it += int(outs[k % len(outs)]["iterations"].sum().item())
        return it

    # W warm-up steps, extended to >= 1.5 s so the GPU's clocks have settled
    # (short timed regions right after start-up measured up to 30% slow)
    t_warm = time.perf_counter()
    n_warm = 0
    if use_stream:
        dec.stream_open(cfg, packed=True, ring_frames=2 * max(F, dec.slots))
        while n_warm < args.warmup or time.perf_counter() - t_warm < 1.5:
            stream_run(args.warmup, lambda k: d_llr, lambda k: d_syn, souts)
            n_warm += args.warmup
    else:
        while n_warm < args.warmup or time.perf_counter() - t_warm < 1.5:
            batch_step()
            int(out["iterations"].sum().item())  # same host read as the timed steps
            n_warm += 1
    torch.cuda.synchronize()
    clocks = ClockSampler(gpu_uuid(torch.cuda.current_device()), args.clock_ms)
    barrier(dist)
    torch.cuda.synchronize()
    clocks.start(not args.no_clocks)
    launches0 = dec.launch_count()
    host0 = time.perf_counter()
    if use_stream:
        # device time: CUDA events on the decoder's own stream (first step)
        # and its output stream (last batch's output copy)
        dec.stream_timer_reset()
        iters_total = stream_run(K, lambda k: d_llr, lambda k: d_syn, souts)
        ms = dec.stream_device_ms()
        torch.cuda.synchronize()
    else:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        iters_total = 0
        for _ in range(K):
            batch_step()
            iters_total += int(out["iterations"].sum().item())  # result gather (host read of the step's outputs)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
    host_ms = (time.perf_counter() - host0) * 1e3
    clock = clocks.stop()
    launches = dec.launch_count() - launches0
    last_out = souts[K - 1] if use_stream else out
    barrier(dist)
    # per-kernel CUDA-event timing: the same K steps again with an event pair
    # around every launch (kept out of the headline timing: the events add
    # host work per launch)
    if use_stream:
        dec.stream_close()
        dec.stream_open(cfg, packed=True, ring_frames=2 * max(F, dec.slots))  # frame-iteration counter from 0
    dec.reset_profile()
    dec.set_profiling(True)
    if use_stream:
        stream_run(K, lambda k: d_llr, lambda k: d_syn, souts)
        dec.stream_close()  # harvests the stream's per-launch events
    else:
        for _ in range(K):
            batch_step()
    torch.cuda.synchronize()
    prof = dec.profile()
    dec.set_profiling(False)
    T = max_over_ranks(ms / 1e3, dist)
    all_iters = sum_over_ranks(float(iters_total), dist)
    edge_updates = all_iters * code.n_edges
    value = edge_updates / T
    reasons = last_out["reasons"].cpu().numpy()
    bits = last_out["bits"].cpu().numpy().view(np.uint32)
    xw = d_x.cpu().numpy().view(np.uint32)
    ok = int(np.sum((reasons == 0) & np.all(bits == xw, axis=1)))
    ok_all = sum_over_ranks(float(ok) * K, dist)
    info_bits = N - M
    d_bar_vnr = all_iters / (F * world * K)

    # ---- roofline of the dominant kernel (check-node update)
    bytes_iter, bytes_check = model_bytes(code)
    lb = layout_bytes(code)
    fi = prof["frame_iterations"]
    peak, peak_kind = measured_peak()
    kern = max(dec.KERNELS, key=lambda k: prof[k]["ms"])
    t_check = prof["check"]["ms"] / 1e3
    t_var = prof["variable"]["ms"] / 1e3
    achieved_check = bytes_check * fi / t_check / 1e9 if t_check > 0 else 0.0
    t_iter = sum(prof[k]["ms"] for k in ("check", "variable", "decide")) / 1e3
    achieved_iter = bytes_iter * fi / t_iter / 1e9 if t_iter > 0 else 0.0
    b_check = lb["check"] * fi / t_check / 1e9 if t_check > 0 else 0.0
    b_var = lb["variable"] * fi / t_var / 1e9 if t_var > 0 else 0.0
    b_step = (lb["check"] + lb["variable"]) * all_iters / T / 1e9 / world
    check_launches = max(prof["check"]["launches"], 1)

    # ---- e2e through the public API with host (pinned) buffers: every step
    # uploads its LLRs + syndromes and reads back bits / iterations / reasons.
    # stream mode: the K batches are submitted back to back from pinned host
    # buffers, outputs land in pinned host buffers, the batch's host result
    # is read after its wait.  batch mode: the upload of step k+1 is staged
    # (bpdec_decoder_stage_inputs) while step k decodes (two host buffer sets).
    in_bytes = F * N * 4 + F * MW * 4
    nbuf = 2
    h_llr = [torch.empty((F, N), dtype=torch.float32, pin_memory=True) for _ in range(nbuf)]
    h_syn = [torch.empty((F, MW), dtype=torch.int32, pin_memory=True) for _ in range(nbuf)]
    for i in range(nbuf):
        h_llr[i].copy_(d_llr)
        h_syn[i].copy_(d_syn)

    def host_out():
        return {"iterations": torch.zeros(F, dtype=torch.int32, pin_memory=True),
                "reasons": torch.zeros(F, dtype=torch.uint8, pin_memory=True),
                "bits": torch.zeros((F, NW), dtype=torch.int32, pin_memory=True)}

    e2e_runs = []
    pipelining = None
    if use_stream:
        h_outs = [host_out() for _ in range(K)]
        dec.stream_open(cfg, packed=True, ring_frames=2 * max(F, dec.slots))
        stream_run(min(K, 4), lambda k: h_llr[k % 2], lambda k: h_syn[k % 2], h_outs)  # warm
        for _rep in range(E2E_RUNS):
            barrier(dist)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_iters = stream_run(K, lambda k: h_llr[k % 2], lambda k: h_syn[k % 2], h_outs)
            torch.cuda.synchronize()
            te = max_over_ranks(time.perf_counter() - t0, dist)
            e2e_runs.append(sum_over_ranks(float(e2e_iters), dist) * code.n_edges / te)
        dec.stream_close()
        pipelining = ("stream mode (bpdec_stream_*): batch k+1's upload and decode start while batch k's tail "
                      "decodes; outputs copied to pinned host buffers as each batch completes")
    else:
        free_b, _ = torch.cuda.mem_get_info()
        staged = 2 * in_bytes < 0.8 * free_b
        h_o = host_out()
        for i in range(nbuf):  # warm the staging buffers
            if staged:
                dec.stage_inputs(h_llr[i], h_syn[i])
            dec.decode_batch(h_llr[i], cfg, syndrome=h_syn[i], packed=True, out=h_o, stream=sptr)
        for _rep in range(E2E_RUNS):
            barrier(dist)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_iters = 0
            if staged:
                dec.stage_inputs(h_llr[0], h_syn[0])
            for k in range(K):
                if staged and k + 1 < K:
                    dec.stage_inputs(h_llr[(k + 1) % 2], h_syn[(k + 1) % 2])
                dec.decode_batch(h_llr[k % 2], cfg, syndrome=h_syn[k % 2], packed=True, out=h_o, stream=sptr)
                e2e_iters += int(h_o["iterations"].numpy().sum())
            torch.cuda.synchronize()
            te = max_over_ranks(time.perf_counter() - t0, dist)
            e2e_runs.append(sum_over_ranks(float(e2e_iters), dist) * code.n_edges / te)
        pipelining = ("upload of step k+1 staged (bpdec_decoder_stage_inputs) during step k" if staged
                      else "none: two staging copies do not fit in device memory")
    e2e_value = float(np.median(e2e_runs))
    h2d = F * N * 4 + F * MW * 4
    d2h = F * NW * 4 + F * 4 + F

    # ---- the other mode's device-resident figure, for the record
    other = None
    if use_stream:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        batch_step()
        torch.cuda.synchronize()
        ev0.record(stream)
        bi = 0
        for _ in range(K):
            batch_step()
            bi += int(out["iterations"].sum().item())
        ev1.record(stream)
        torch.cuda.synchronize()
        tb = max_over_ranks(ev0.elapsed_time(ev1) / 1e3, dist)
        other = {"mode": "batch (one blocking bpdec_decode_batch per step; each batch ends in its VNR tail)",
                 "value": sum_over_ranks(float(bi), dist) * code.n_edges / tb, "ms_per_step": 1e3 * tb / K}
    else:
        souts = [dev_out() for _ in range(K)]
        dec.stream_open(cfg, packed=True, ring_frames=2 * max(F, dec.slots))
        stream_run(min(K, 4), lambda k: d_llr, lambda k: d_syn, souts)
        dec.stream_timer_reset()
        si = stream_run(K, lambda k: d_llr, lambda k: d_syn, souts)
        ts = max_over_ranks(dec.stream_device_ms() / 1e3, dist)
        dec.stream_close()
        other = {"mode": "stream (the K batches back to back through bpdec_stream_*, device-resident inputs)",
                 "value": sum_over_ranks(float(si), dist) * code.n_edges / ts, "ms_per_step": 1e3 * ts / K}

    # ---- VNR vs PCE comparison (one PCE batch, not part of the timed metric)
    pce = None
    if not args.no_pce_compare:
        cfg_p = P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=False, q_mode=Q_ABS)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dec.decode_batch(d_llr, cfg_p, syndrome=d_syn, packed=True, out=out, stream=sptr)
        e1.record(stream)
        torch.cuda.synchronize()
        tp_s = max_over_ranks(e0.elapsed_time(e1) / 1e3, dist)
        pit = sum_over_ranks(float(out["iterations"].sum().item()), dist)
        prs = out["reasons"].cpu().numpy()
        pbits = out["bits"].cpu().numpy().view(np.uint32)
        pok = sum_over_ranks(float(np.sum((prs == 0) & np.all(pbits == xw, axis=1))), dist)
        pce = {"d_bar": pit / (F * world), "edge_updates_per_s": pit * code.n_edges / tp_s,
               "decoded_info_bits_per_s": pok * info_bits / tp_s,
               "frames_per_s": F * world / tp_s, "fer": 1.0 - pok / (F * world)}

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            if oracle.reference_available():
                threads = os.cpu_count() or 1
                nf = args.cpu_frames or threads
                llr_h = d_llr[:nf].cpu().numpy()
                xh = P.unpack_bits(xw[:nf], N)
                leq = (llr_h * (1 - 2 * xh.astype(np.float32))).astype(np.float64)
                cpu_reference_time(code, leq[:1], w.d_max, 1)  # first touch warm-up
                dt, it, _ = cpu_reference_time(code, leq, w.d_max, threads)
                cpu = {"value": it * code.n_edges / dt, "unit": UNIT, "cores": threads, "kind": "reference",
                       "cpu_model": cpu_model(),
                       "sample": f"{nf} frames of {w.name} (beta={beta if brange is None else brange}, VNR+PCE, "
                                 f"D_max={w.d_max}), "
                                 f"one reference BpDecoder per thread, {dt:.1f} s"}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    # ---- live DRAM traffic of k_check (ncu, child process; rank 0, N=1)
    traffic, traffic_note = None, "not measured (N>1 or --no-traffic)"
    if rank == 0 and world == 1 and not args.no_traffic:
        del dec
        torch.cuda.empty_cache()
        traffic, traffic_note = measure_traffic(args)

    if rank == 0:
        emit({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / K, "higher_is_better": True,
            "host_ms_per_step": host_ms / K, "warmup_steps_run": n_warm,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded BASELINE generator, device-generated frames)",
            "config": {"workload": w.name, "frames_per_gpu": F, "slots": slots,
                       "beta": beta if brange is None else list(brange),
                       "d_max": w.d_max, "et": "vnr+pce", "q_mode": "abs (syndrome mode)",
                       "mode": ("stream: the K batches submitted back to back through bpdec_stream_*"
                                if use_stream else "batch: one blocking bpdec_decode_batch per step"),
                       "parallelism": f"frame-shard x{world}",
                       "l2": "working set (~0.7 GB per GPU) >> 126 MB L2; no flush needed"},
            "decoded_info_bits_per_s": ok_all * info_bits / T,
            "processed_info_bits_per_s": F * world * K * info_bits / T,
            "frames_per_s": F * world * K / T,
            "fer": 1.0 - ok / F,
            "d_bar_vnr": d_bar_vnr,
            "other_mode": other,
            "pce": pce,
            "vnr_vs_pce": None if pce is None else {
                "iteration_gain": pce["d_bar"] / d_bar_vnr,
                "frame_throughput_gain": (F * world * K / T) / pce["frames_per_s"]},
            "roofline": {"bound": "hbm", "kernel": "k_check", "achieved": achieved_check, "peak": peak,
                         "unit": "GB/s", "frac": achieved_check / peak,
                         "traffic": None if traffic is None else traffic["bytes_per_launch"],
                         "traffic_measured": traffic if traffic is not None else traffic_note,
                         "peak_kind": peak_kind,
                         "bytes_model": "model A (BASELINE.md §2): check pass = 8E per frame-iteration",
                         "note": ("model A counts naive per-edge messages; this layout moves fewer bytes (model_b, "
                                  "traffic), so a model-A frac above 1 is possible -- dram_frac is the kernel's "
                                  "measured DRAM bytes over its CUDA-event time, the real utilisation"),
                         "dram_achieved": (None if traffic is None or t_check <= 0 else
                                           traffic["bytes_per_frame_iteration"] * fi / t_check / 1e9),
                         "dram_frac": (None if traffic is None or t_check <= 0 else
                                       traffic["bytes_per_frame_iteration"] * fi / t_check / 1e9 / peak),
                         "model_b": {"what": "bytes this layout moves per frame-iteration (DESIGN.md §3)",
                                     "check_bytes": lb["check"], "variable_bytes": lb["variable"],
                                     "check_achieved": b_check, "check_frac": b_check / peak,
                                     "variable_achieved": b_var, "variable_frac": b_var / peak,
                                     "step_achieved": b_step, "step_frac": b_step / peak,
                                     "check_traffic_vs_model_b": (None if traffic is None else
                                                                  traffic["bytes_per_frame_iteration"] / lb["check"])},
                         "iteration_achieved": achieved_iter, "iteration_frac": achieved_iter / peak,
                         "dominant_by_time": kern,
                         "kernel_ms": {k: prof[k]["ms"] for k in P.BatchDecoder.KERNELS},
                         "check_launches": check_launches,
                         "check_us_per_launch": 1e6 * t_check / check_launches,
                         "frame_iterations": fi},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "runs": e2e_runs, "note": f"median of {E2E_RUNS} timed runs of {K} steps",
                    "pipelining": pipelining},
            "gpu_launches": launches,
            "clocks": clock,
        })
    barrier(dist)
    if dist is not None:
        dist.destroy_process_group()


def run_multi(args):
    """Strong scaling inside one process: the
    K x F frames of the run are decoded by bpdec_multi_decode_batch over
    --gpus devices (one decoder and host thread per GPU, dynamic chunk
    queue, outputs gathered into the caller's host buffers).  Timed with the
    host clock from the call to its return (the API's own contract: inputs
    and outputs in host memory), after a warm-up call."""
    import torch
    import paper_2507_03509_b200 as P
    from paper_2507_03509_b200.decoder import Q_ABS
    devices = ([int(x) for x in args.multi_devices.split(",")] if args.multi_devices
               else list(range(args.gpus)))
    ng = len(devices)
    if torch.cuda.device_count() <= max(devices):
        raise SystemExit(f"bench --multi: devices {devices} requested, {torch.cuda.device_count()} visible")
    w = P.WORKLOADS[args.workload]
    code = w.make_code()
    F = args.frames or FRAMES[args.workload]
    total = F * max(1, args.steps)
    N, M = code.n_vars, code.n_checks
    MW, NW = (M + 31) // 32, (N + 31) // 32
    beta, brange = workload_beta(args)
    slots = args.slots or min(F, 512)
    gen = P.BatchDecoder(code, device=0, max_slots=32)
    h_llr = torch.empty((total, N), dtype=torch.float32, pin_memory=True)
    h_syn = torch.empty((total, MW), dtype=torch.int32, pin_memory=True)
    step = 256
    for f0 in range(0, total, step):
        n = min(step, total - f0)
        d_llr, d_syn, _ = make_frames(P, gen, code, args, n, f0, 0)
        h_llr[f0:f0 + n].copy_(d_llr)
        h_syn[f0:f0 + n].copy_(d_syn)
        del d_llr, d_syn
    del gen
    torch.cuda.empty_cache()
    cfg = P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=True, q_mode=Q_ABS)
    m = P.MultiDecoder(code, devices, slots_per_decoder=slots)
    h_out = {"iterations": torch.zeros(total, dtype=torch.int32, pin_memory=True),
             "reasons": torch.zeros(total, dtype=torch.uint8, pin_memory=True),
             "bits": torch.zeros((total, NW), dtype=torch.int32, pin_memory=True)}
    m.decode_batch(h_llr, cfg, syndrome=h_syn, packed=True, out=h_out)  # warm-up: the full batch once
    runs = []
    for _rep in range(E2E_RUNS):
        t0 = time.perf_counter()
        m.decode_batch(h_llr, cfg, syndrome=h_syn, packed=True, out=h_out)
        runs.append(time.perf_counter() - t0)
    T = float(np.median(runs))
    it = float(h_out["iterations"].numpy().sum())
    value = it * code.n_edges / T
    emit({"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": len(set(devices)), "steps": args.steps,
          "warmup": 1, "devices": devices,
          "ms_per_step": 1e3 * T / max(1, args.steps), "higher_is_better": True, "scaling": "strong",
          "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded BASELINE generator)",
          "config": {"workload": w.name, "frames_total": total, "slots_per_gpu": slots,
                     "beta": beta if brange is None else list(brange), "d_max": w.d_max, "et": "vnr+pce",
                     "parallelism": f"bpdec_multi x{ng} on devices {devices} (dynamic chunk queue, host gather)"},
          "frames_per_decoder": m.last_frames_per_decoder.tolist(), "d_bar_vnr": it / total,
          "runs_s": runs, "timing_note": f"median of {E2E_RUNS} calls after a full-size warm-up call",
          "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": F * (N + MW) * 4,
                  "d2h_bytes_per_step": F * (NW * 4 + 5)},
          "timing": "host clock around bpdec_multi_decode_batch (host buffers in and out)"})
    m.close()


def main():
    args = parse()
    if args.traffic_probe:
        return traffic_probe(args)
    if args.ref_inputs is not None:
        return write_reference_inputs(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.multi:
        return run_multi(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    run_ours(args)


if __name__ == "__main__":
    main()
