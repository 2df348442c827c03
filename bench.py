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
FRAMES = {"cfg1": 16, "cfg2": 64, "cfg3": 32, "cfg4": 512, "cfg5": 1024}


def workload_beta(args):
    """(beta, beta_range) for the workload: fixed beta, or a per-frame range."""
    if args.workload == "cfg5" and args.beta is None:
        return None, (0.92, 1.0)
    if args.beta is not None:
        return args.beta, None
    return (0.98 if args.workload == "cfg3" else 0.95), None


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
    return ap.parse_args()


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
def run_reference(args):
    """Rank 0 alone times the reference CPU decoder; other ranks exit."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    import paper_2507_03509_b200 as P
    w = P.WORKLOADS[args.workload]
    import oracle
    if not oracle.reference_available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/libetdec_ref.so not built (needs /root/reference)"})
        return
    code = w.make_code()
    threads = os.cpu_count() or 1
    frames = args.cpu_frames or threads
    beta, brange = workload_beta(args)
    if brange is None:
        llr, x, _ = P.sample_frames(code, P.snr_for_beta(beta, code.rate()), P.FRAME_SEED, 0, frames)
    else:
        llr, x, _, _ = P.sample_frames_beta(code, brange[0], brange[1], P.FRAME_SEED, 0, frames)
    leq = (llr * (1 - 2 * x.astype(np.float32))).astype(np.float64)
    times, iters = [], []
    for k in range(args.warmup + args.steps):
        dt, it, _ = cpu_reference_time(code, leq, w.d_max, threads)
        if k >= args.warmup:
            times.append(dt)
            iters.append(it)
    T = float(np.sum(times))
    value = float(np.sum(iters)) * code.n_edges / T
    sample = (f"{frames} frames of {w.name} (beta={beta if brange is None else brange}, VNR+PCE, "
              f"D_max={w.d_max}) per step, "
              f"all-zero-equivalent inputs L*(1-2x), s=0 (the reference's semantics)")
    emit({"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
          "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times),
          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
          "data": "synthetic (seeded BASELINE generator)",
          "config": {"workload": w.name, "frames_per_step": frames, "beta": beta if brange is None else list(brange),
                     "d_max": w.d_max,
                     "et": "vnr+pce", "threads": threads},
          "d_bar": float(np.sum(iters)) / (frames * len(times)),
          "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                           "sample": sample},
          "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})


# ------------------------------------------------------------- our arm --
def run_ours(args):
    rank, world, local, dist = dist_setup(args.gpus)
    import torch
    import paper_2507_03509_b200 as P
    from paper_2507_03509_b200.decoder import Q_ABS

    torch.cuda.set_device(local)
    w = P.WORKLOADS[args.workload]
    code = w.make_code()
    F = args.frames or FRAMES[args.workload]
    slots = args.slots or min(F, 512)
    beta, brange = workload_beta(args)
    dec = P.BatchDecoder(code, device=local, max_slots=slots)
    snr = P.snr_for_beta(beta, code.rate()) if brange is None else 0.0
    # weak scaling: rank r owns global frames [r*F, (r+1)*F)
    first = rank * F
    N, M = code.n_vars, code.n_checks
    MW, NW = (M + 31) // 32, (N + 31) // 32
    stream = torch.cuda.Stream(device=local)
    sptr = stream.cuda_stream
    d_llr = torch.empty((F, N), dtype=torch.float32, device="cuda")
    d_syn = torch.empty((F, MW), dtype=torch.int32, device="cuda")
    d_x = torch.empty((F, NW), dtype=torch.int32, device="cuda")
    dec.sample_frames_device(snr, P.FRAME_SEED, first, F, d_llr, d_syn, d_x, stream=sptr, beta_range=brange)
    out = {"iterations": torch.zeros(F, dtype=torch.int32, device="cuda"),
           "reasons": torch.zeros(F, dtype=torch.uint8, device="cuda"),
           "bits": torch.zeros((F, NW), dtype=torch.int32, device="cuda")}
    cfg = P.DecodeConfig(d_max=w.d_max, use_pce=True, use_vnr=True, q_mode=Q_ABS)

    def step():
        return dec.decode_batch(d_llr, cfg, syndrome=d_syn, packed=True, out=out, stream=sptr)

    # W warm-up steps, extended to >= 1.5 s so the GPU's clocks have settled
    # (short timed regions right after start-up measured up to 30% slow)
    t_warm = time.perf_counter()
    n_warm = 0
    while n_warm < args.warmup or time.perf_counter() - t_warm < 1.5:
        step()
        int(out["iterations"].sum().item())  # same host read as the timed steps (loads torch's kernel once)
        n_warm += 1
    torch.cuda.synchronize()
    clocks = ClockSampler(gpu_uuid(torch.cuda.current_device()), args.clock_ms)
    barrier(dist)
    torch.cuda.synchronize()
    clocks.start(not args.no_clocks)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches0 = dec.launch_count()
    host0 = time.perf_counter()
    ev0.record(stream)
    iters_total = 0
    for _ in range(args.steps):
        r = step()
        iters_total += int(out["iterations"].sum().item())  # result gather (host read of the step's outputs)
    ev1.record(stream)
    torch.cuda.synchronize()
    host_ms = (time.perf_counter() - host0) * 1e3
    clock = clocks.stop()
    launches = dec.launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    barrier(dist)
    # per-kernel CUDA-event timing: the same K steps again with an event pair
    # around every launch (kept out of the headline timing: the events add
    # host work per launch)
    dec.reset_profile()
    dec.set_profiling(True)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    prof = dec.profile()
    dec.set_profiling(False)
    T = max_over_ranks(ms / 1e3, dist)
    all_iters = sum_over_ranks(float(iters_total), dist)
    edge_updates = all_iters * code.n_edges
    value = edge_updates / T
    reasons = out["reasons"].cpu().numpy()
    bits = out["bits"].cpu().numpy().view(np.uint32)
    xw = d_x.cpu().numpy().view(np.uint32)
    ok = int(np.sum((reasons == 0) & np.all(bits == xw, axis=1)))
    ok_all = sum_over_ranks(float(ok) * args.steps, dist)
    info_bits = N - M
    d_bar_vnr = all_iters / (F * world * args.steps)

    # ---- roofline of the dominant kernel (check-node update)
    bytes_iter, bytes_check = model_bytes(code)
    fi = prof["frame_iterations"]
    peak, peak_kind = measured_peak()
    kern = max(dec.KERNELS, key=lambda k: prof[k]["ms"])
    t_check = prof["check"]["ms"] / 1e3
    achieved_check = bytes_check * fi / t_check / 1e9 if t_check > 0 else 0.0
    t_iter = sum(prof[k]["ms"] for k in ("check", "variable", "decide")) / 1e3
    achieved_iter = bytes_iter * fi / t_iter / 1e9 if t_iter > 0 else 0.0
    # model B: the bytes this layout must move per frame-iteration
    dims = code
    traffic = None
    tp = os.path.join(ROOT, "profiles", "check_kernel_dram_bytes.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                tj = json.load(f)
            if tj.get("workload") == w.name:
                traffic = tj.get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None

    # ---- e2e through the public API with host (pinned) buffers: every step
    # uploads its LLRs + syndromes and reads back bits / iterations / reasons.
    # The upload of step k+1 is staged (bpdec_decoder_stage_inputs) before
    # step k decodes, so it overlaps the decode (two host buffer sets) — when
    # two staging copies fit in device memory; otherwise each step uploads
    # inside the decode call.
    in_bytes = F * N * 4 + F * MW * 4
    free_b, _ = torch.cuda.mem_get_info()
    staged = 2 * in_bytes < 0.8 * free_b
    nbuf = 2 if staged else 1
    h_llr = [torch.empty((F, N), dtype=torch.float32, pin_memory=True) for _ in range(nbuf)]
    h_syn = [torch.empty((F, MW), dtype=torch.int32, pin_memory=True) for _ in range(nbuf)]
    for i in range(nbuf):
        h_llr[i].copy_(d_llr)
        h_syn[i].copy_(d_syn)
    h_out = {"iterations": torch.zeros(F, dtype=torch.int32, pin_memory=True),
             "reasons": torch.zeros(F, dtype=torch.uint8, pin_memory=True),
             "bits": torch.zeros((F, NW), dtype=torch.int32, pin_memory=True)}
    for i in range(nbuf):  # warm the staging buffers
        if staged:
            dec.stage_inputs(h_llr[i], h_syn[i])
        dec.decode_batch(h_llr[i], cfg, syndrome=h_syn[i], packed=True, out=h_out, stream=sptr)
    # the K-step timed region is short (~0.25 s for cfg2) and a host hiccup
    # shows in it: it runs three times and the median is reported (all runs
    # are listed in the JSON line)
    K = max(1, args.steps)
    e2e_runs = []
    for _rep in range(3):
        barrier(dist)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_iters = 0
        if staged:
            dec.stage_inputs(h_llr[0], h_syn[0])
        for k in range(K):
            if staged and k + 1 < K:
                dec.stage_inputs(h_llr[(k + 1) % 2], h_syn[(k + 1) % 2])
            dec.decode_batch(h_llr[k % nbuf], cfg, syndrome=h_syn[k % nbuf], packed=True, out=h_out, stream=sptr)
            e2e_iters += int(h_out["iterations"].numpy().sum())
        torch.cuda.synchronize()
        te = max_over_ranks(time.perf_counter() - t0, dist)
        e2e_runs.append(sum_over_ranks(float(e2e_iters), dist) * code.n_edges / te)
    e2e_value = float(np.median(e2e_runs))
    h2d = F * N * 4 + F * MW * 4
    d2h = F * NW * 4 + F * 4 + F

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
               "frames_per_s": F * world / tp_s}

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
                       "sample": f"{nf} frames of {w.name} (beta={beta if brange is None else brange}, VNR+PCE, "
                                 f"D_max={w.d_max}), "
                                 f"one reference BpDecoder per thread, {dt:.1f} s"}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        emit({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "host_ms_per_step": host_ms / args.steps, "warmup_steps_run": n_warm,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded BASELINE generator, device-generated frames)",
            "config": {"workload": w.name, "frames_per_gpu": F, "slots": dec.slots,
                       "beta": beta if brange is None else list(brange),
                       "d_max": w.d_max, "et": "vnr+pce", "q_mode": "abs (syndrome mode)",
                       "parallelism": f"frame-shard x{world}",
                       "l2": "working set (~0.7 GB per GPU) >> 126 MB L2; no flush needed"},
            "decoded_info_bits_per_s": ok_all * info_bits / (T * args.steps) * args.steps,
            "processed_info_bits_per_s": F * world * args.steps * info_bits / T,
            "frames_per_s": F * world * args.steps / T,
            "d_bar_vnr": d_bar_vnr,
            "pce": pce,
            "vnr_vs_pce": None if pce is None else {
                "iteration_gain": pce["d_bar"] / d_bar_vnr,
                "frame_throughput_gain": (F * world * args.steps / T) / pce["frames_per_s"]},
            "roofline": {"bound": "hbm", "kernel": "k_check", "achieved": achieved_check, "peak": peak,
                         "unit": "GB/s", "frac": achieved_check / peak, "traffic": traffic,
                         "peak_kind": peak_kind,
                         "bytes_model": "model A (BASELINE.md §2): check pass = 8E per frame-iteration",
                         "iteration_achieved": achieved_iter, "iteration_frac": achieved_iter / peak,
                         "dominant_by_time": kern,
                         "kernel_ms": {k: prof[k]["ms"] for k in dec.KERNELS},
                         "frame_iterations": fi},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "runs": e2e_runs, "note": f"median of 3 timed runs of {K} steps",
                    "pipelining": ("upload of step k+1 staged (bpdec_decoder_stage_inputs) during step k" if staged
                                   else "none: two staging copies do not fit in device memory")},
            "gpu_launches": launches,
            "clocks": clock,
        })
    barrier(dist)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
