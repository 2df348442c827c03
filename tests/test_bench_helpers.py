"""Host-side pieces of bench.py (CPU): the model-B byte counts the roofline
reports, the reference arm's input files, the per-workload beta, and the
frame sharding."""
import argparse
import json
import os
import sys

import numpy as np

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_layout_bytes_cfg2(P):
    """Model B for the BASELINE cfg2 code: check pass
    8 (E_hi - n11) + 4 N1, variable pass 4 E_hi + 8 N_V."""
    code = P.WORKLOADS["cfg2"].make_code()
    lb = bench.layout_bytes(code)
    assert (lb["e_hi"], lb["n_deg1"], lb["n_v"]) == (1494222, 786432, 262144)
    assert lb["check"] == 8 * (lb["e_hi"] - lb["n11"]) + 4 * lb["n_deg1"]
    assert lb["variable"] == 4 * lb["e_hi"] + 8 * lb["n_v"]
    per_edge = (lb["check"] + lb["variable"]) / code.n_edges
    assert 8.5 < per_edge < 9.0  # ~8.8 B per edge-update vs 17.95 for model A
    a_iter, a_check = bench.model_bytes(code)
    assert a_check == 8 * code.n_edges and abs(a_iter / code.n_edges - 17.95) < 0.01


def test_reference_inputs_roundtrip(P, tmp_path):
    """--impl reference: the child writes the code and the all-zero-equivalent
    frames; they equal the package's own generator's output."""
    args = argparse.Namespace(workload="cfg1", cpu_frames=3, beta=None, ref_inputs=str(tmp_path))
    bench.write_reference_inputs(args)
    meta = json.load(open(os.path.join(tmp_path, "meta.json")))
    ptr = np.load(os.path.join(tmp_path, "check_ptr.npy"))
    var = np.load(os.path.join(tmp_path, "check_vars.npy"))
    leq = np.load(os.path.join(tmp_path, "llr.npy"))
    code = P.WORKLOADS["cfg1"].make_code()
    p0, v0 = code.csr()
    assert np.array_equal(ptr, p0) and np.array_equal(var, v0)
    assert meta["frames"] == 3 and meta["d_max"] == 200 and leq.shape == (3, code.n_vars)
    llr, x, _ = P.sample_frames(code, P.snr_for_beta(meta["beta"], code.rate()), P.FRAME_SEED, 0, 3)
    assert np.array_equal(leq, (llr * (1 - 2 * x.astype(np.float32))).astype(np.float64))


def test_workload_beta_defaults():
    ns = lambda w, b=None: argparse.Namespace(workload=w, beta=b)  # noqa: E731
    assert bench.workload_beta(ns("cfg2")) == (0.96, None)      # middle of configs[1]'s grid
    assert bench.workload_beta(ns("cfg3")) == (0.98, None)
    assert bench.workload_beta(ns("cfg5")) == (None, (0.92, 1.0))
    assert bench.workload_beta(ns("met")) == (0.87, None)       # inside the waterfall
    assert bench.workload_beta(ns("cfg2", 0.9)) == (0.9, None)


def test_sweep_tables_render_committed_profiles():
    """scripts/sweep_tables.py renders DESIGN.md's ET tables from the
    committed sweep JSONs (one row per beta, FER / D-bar columns present)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prof = os.path.join(root, "profiles", "r2")
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "sweep_tables.py"),
                          os.path.join(prof, "et_sweep_cfg2.json"), os.path.join(prof, "et_sweep_cfg5.json")],
                         capture_output=True, text=True, check=True).stdout
    rows = [l for l in out.splitlines() if l.startswith("| 0.") or l.startswith("| cfg5")]
    assert len(rows) == 14 and "| 0.96 |" in out
    met = subprocess.run([sys.executable, os.path.join(root, "scripts", "sweep_tables.py"), "--met",
                          os.path.join(prof, "et_sweep_met.json")], capture_output=True, text=True, check=True).stdout
    assert met.count("\n| 0.") == 8 and "beta_opt" in met
