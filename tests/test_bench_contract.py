"""bench.py's JSON line keeps the driver's contract.

not gpu: the reference arm (the oracle on the host cores, one full batch per step)
prints one JSON line with the keys the driver reads and reports the steps it timed.
gpu: the product arm's line carries the roofline, clocks, e2e, gpu_launches and
cpu_baseline objects (c1q3, a short run)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "c1q3", "--steps", "2", "--warmup", "1", "--ref-budget", "30"], 600)
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "queries/s" and d["higher_is_better"] is True
    assert 1 <= d["steps"] <= 2 and d["config"]["requested"] == {"steps": 2, "warmup": 1}
    # the timed steps are whole batches: value = queries per step / time per step
    assert abs(d["value"] - d["config"]["queries_per_step"] / (d["ms_per_step"] / 1e3)) < 1e-6 * d["value"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_product_line():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    d = _run(["--config", "c1q3", "--steps", "2000", "--warmup", "3", "--no-cpu"], 900)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert k in d, k
    assert d["steps"] == 2000 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["config"]["workload"] == "c1q3"
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert 0 < r["frac"] < 1.0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["gpu_launches"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_committed_c5_sweep_is_clocked_and_complete():
    """The committed c5 evidence (profiles/r02/r67/c5_all.jsonl, BASELINE.json configs[4]):
    every ephdc_inputs.c5_points point is present for NTT and MAC, every line carries a
    clock record with samples, and no line saw a thermal / hardware slowdown."""
    import ephdc_inputs as inp
    path = os.path.join(ROOT, "profiles", "r02", "r67", "c5_all.jsonl")
    rows = [json.loads(l) for l in open(path) if l.strip().startswith("{")]
    ntt = {(r["log2N"], r["L"], r["bits"], r["word_bits"] // 8) for r in rows if "ntt_fwd" in r}
    mac = {(r["log2N"], r["L"], r["bits"], r["word_bits"] // 8) for r in rows if r.get("op") == "mac"}
    want = {tuple(p[:4]) for p in inp.c5_points("all")}
    assert ntt == want and mac == want
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    for r in rows:
        c = r["clocks"]
        assert c["samples"] >= 1 and c["sm_mhz"] and not (bad & set(c["reasons"])), r
