"""bench.py's GPU arm keeps the driver's JSON contract (one line; roofline, cpu_baseline, e2e,
gpu_launches, clocks; the m sweep) -- run at a reduced n_local so the test takes seconds.
The driver's own runs use the defaults (config 2, n_local = 1e8)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpu_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--n-local", "2097152", "--steps", "3",
                        "--warmup", "3", "--cpu-n", "100000"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    L = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
                "gpu_launches", "clocks", "sweep"):
        assert key in L, key
    assert L["n_gpus"] == 1 and L["steps"] == 3 and L["warmup"] >= 3 and L["higher_is_better"] is False
    assert L["dtype"] == "f64" and L["scaling"] == "weak" and L["config"]["workload"]
    assert abs(L["value"] - 1e3 * L["ms_per_step"]) <= 1e-6 * L["value"]
    rf = L["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) <= 1e-9
    assert 0.1 < rf["frac"] < 1.3
    cb = L["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > L["value"] and cb["sample"]
    e2e = L["e2e"]
    assert e2e["h2d_bytes_per_step"] == 8 * 2097152 and e2e["d2h_bytes_per_step"] == 8 * 2097152
    assert e2e["value"] > 0
    assert L["gpu_launches"] == 3 * L["steps"]   # DCGS-2: K1, K2, K4 per step
    assert "sm_mhz" in L["clocks"] and "reasons" in L["clocks"]
    assert {f"{v}_m{m}" for v in ("dcgs2", "icwy", "cgs2", "mgs", "icwy_small") for m in (5, 10, 20, 50)} <= set(L["sweep"])


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_gpu_arm_json_line_torchrun():
    """The driver's N > 1 launch (torchrun, one rank per GPU): rank 0 prints one line with the
    whole-job value, the max-over-ranks timing and the per-exchange latency curve."""
    world = min(torch.cuda.device_count(), 4)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", "29561", os.path.join(ROOT, "bench.py"),
                        "--gpus", str(world), "--n-local", "2097152", "--steps", "3", "--warmup", "3", "--no-sweep"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    L = json.loads(lines[0])
    assert L["n_gpus"] == world and L["scaling"] == "weak"
    assert "exchange_latency" in L and L["e2e"]["value"] > 0 and L["gpu_launches"] == 3 * L["steps"]
    assert all(v["fused_us"] > 0 and v["nccl_us"] > 0 for v in L["exchange_latency"].values())
