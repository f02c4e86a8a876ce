"""bench.py's JSON contract: the reference arm on the CPU (the numpy oracle
port), our arm on a GPU (roofline, launches, e2e and clock keys)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--config", "llama7b_p6000_b64"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["workload"] == "llama7b_p6000_b64"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    # one step of this arm is one sampled layer, and the line says so
    assert d["extrapolated"] is True and d["ms_per_step"] == d["layer_ms"]
    assert d["steps"] * d["ms_per_step"] / 1e3 <= d["wall_s"]


@pytest.mark.gpu
def test_ours_arm_line():
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                          "--config", "llama7b_p6000_b64", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0.3 < r["frac"] < 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["gpu_launches"] == 3 * (32 * 3 + 1)
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and d["n_gpus"] == 1 and d["scaling"] == "weak"
    assert d["value"] > 1000
    # the timed configuration is the verified one
    p = d["parity"]
    assert p["pass"] and p["layers"] == [0, 31] and p["max_abs"] <= 2e-2 and p["mean_rel_f32"] <= 1e-3
    assert 0.3 < r["frac_isolated"] <= r["frac"] * 1.05 and r["layer_us_isolated"] > 0


@pytest.mark.gpu
def test_two_rank_torchrun_on_one_gpu():
    """bench.py under torchrun with 2 ranks sharing cuda:0: one engine per
    rank, no collective on the data path (gloo only for the barrier and the
    max-over-ranks timing), rank 0 prints one line with the whole-job rows;
    the strong-scaling config deals the 8 nested apps over the ranks."""
    for config, rows in (("llama7b_p6000_b64", 128), ("nested_smoke_8apps", 512)):
        res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                              "--master-addr", "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "bench.py"),
                              "--gpus", "2", "--steps", "3", "--warmup", "3", "--config", config, "--no-e2e",
                              "--no-check", "--no-isolated", "--no-cpu-baseline"],
                             capture_output=True, text=True, timeout=900, cwd=ROOT)
        assert res.returncode == 0, res.stderr[-3000:]
        lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
        assert len(lines) == 1, res.stdout[-2000:]
        d = json.loads(lines[0])
        assert d["n_gpus"] == 2 and d["rows_total"] == rows and d["value"] > 0
        assert d["scaling"] == ("strong" if config.startswith("nested") else "weak")
