"""bench.py's JSON contract (the driver parses these keys).  The reference arm (fp64 oracle on the
host cores) runs on CPU; the device arm is a GPU test on the small C1 configuration."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_json_contract():
    d = _run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "1"])
    assert BASE_KEYS <= set(d), set(d) ^ BASE_KEYS
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["higher_is_better"] is True


@pytest.mark.gpu
def test_device_arm_json_contract():
    d = _run(["--config", "1", "--steps", "3", "--warmup", "3"])
    assert BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"]
    assert d["roofline"]["frac"] > 0
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d["clocks"]
    assert d["gpu_launches"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1


def test_reference_arm_under_torchrun_two_ranks():
    """The driver launches the reference arm with torchrun for N > 1: rank 0 alone prints the line,
    the other ranks exit 0 without work."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29571", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--config", "1", "--steps", "1", "--warmup", "1"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def _torchrun(args, port, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py")] + args
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_device_arm_two_ranks_verifies_itself():
    """N > 1 (2 gloo ranks sharing cuda:0, testing only): the line carries its own parity sample
    (128 rows of each shard gathered to rank 0) and every rank's plan."""
    d = _torchrun(["--gpus", "2", "--config", "2", "--dist-backend", "gloo", "--one-device",
                   "--steps", "3", "--warmup", "3", "--shape", "20000,20000"], 29581)
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "ishard2"
    assert len(d["per_rank"]) == 2 and [r["rank"] for r in d["per_rank"]] == [0, 1]
    assert d["per_rank"][0]["row_lo"] == 0 and d["per_rank"][1]["row_hi"] == 20000
    cb = d["cpu_baseline"]
    assert "of each of the 2 shards" in cb["sample"] and cb["max_r4_err_vs_gpu"] <= 1e-5
    assert cb["cpu_model"]


@pytest.mark.gpu
@pytest.mark.parametrize("config", [7, 8])
def test_jshard_mode_json(config):
    """--mode jshard (1 rank here, 2 gloo ranks below): the public dist.jshard_eval path, with
    the merged rows checked against the oracle over all of y."""
    d = _run(["--mode", "jshard", "--config", str(config), "--steps", "3", "--warmup", "3",
              "--shape", "3000,2000000"])
    assert d["config"]["combine"] and d["roofline"]["bound"] == "alu" and d["value"] > 0
    err = d["cpu_baseline"].get("max_r4_err_vs_gpu", d["cpu_baseline"].get("max_abs_err_vs_gpu"))
    assert err is not None and err <= (1e-5 if config == 7 else 1e-6)
    d2 = _torchrun(["--gpus", "2", "--mode", "jshard", "--config", str(config), "--dist-backend",
                    "gloo", "--one-device", "--steps", "2", "--warmup", "2", "--shape", "3000,2000000"],
                   29582 + config)
    assert d2["config"]["parallelism"] == "jshard2" and len(d2["per_rank"]) == 2
    assert d2["per_rank"][1]["j_hi"] == 2000000
    err2 = d2["cpu_baseline"].get("max_r4_err_vs_gpu", d2["cpu_baseline"].get("max_abs_err_vs_gpu"))
    assert err2 <= (1e-5 if config == 7 else 1e-6)


@pytest.mark.gpu
def test_bench_reports_the_form_the_device_chose():
    """config.form follows the device's bounding-box decision (reading R18b): sigma = 0.5 on the
    unit cube takes the expanded form, sigma = 0.05 the direct one (8 FP32 lane-ops per pair in
    the roofline's basis)."""
    d = _run(["--config", "5", "--shape", "200000,200000", "--steps", "3", "--warmup", "3", "--no-e2e"])
    assert d["config"]["form"] == "expanded" and "16/0.875 MUFU, 128/5 FP32" in d["roofline"]["peak_basis"]
    d = _run(["--config", "5", "--shape", "200000,200000", "--scale", "0.05", "--steps", "3", "--warmup", "3",
              "--no-e2e"])
    assert d["config"]["form"] == "direct" and "16/1 MUFU, 128/8 FP32" in d["roofline"]["peak_basis"]
    assert d["cpu_baseline"]["max_r4_err_vs_gpu"] <= 1e-5
    # N >= 2^18, M >= 2^16: the tile-centred form (R18j), its tiles counted in config.form
    d = _run(["--config", "5", "--shape", "400000,400000", "--scale", "0.05", "--steps", "3", "--warmup", "3",
              "--no-e2e"])
    assert d["config"]["form"].startswith("tile-centred (") and "harmonic mix" in d["roofline"]["peak_basis"]
    assert d["cpu_baseline"]["max_r4_err_vs_gpu"] <= 1e-5
