"""The bench.py JSON-line contract (keys the driver and the judge read).

The reference arm runs here on CPU (the oracle port of the reference algorithm on a
bounded sample); the GPU arm is a `-m gpu` test on the smallest BASELINE video config.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert lines, r.stdout[-2000:]
    return json.loads(lines[-1])


def _common(d):
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "e2e"):
        assert key in d, key
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["higher_is_better"] is True
    assert "workload" in d["config"]


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "wan13b_480p"], 600)
    _common(d)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]


@pytest.mark.gpu
def test_gpu_arm_contract():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--steps", "3", "--warmup", "3", "--no-cpu", "--config", "wan13b_480p"], 900)
    _common(d)
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "tensor") and rf["unit"] in ("GB/s", "TFLOP/s")
    assert 0 < rf["frac"] < 1 and abs(rf["achieved"] / rf["peak"] - rf["frac"]) < 1e-9
    assert d["gpu_launches"] > 0
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    e2e = d["e2e"]
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0 and 0 < e2e["value"] < d["value"]


def test_reference_arm_two_ranks():
    """--gpus 2 without torchrun: bench.py starts two ranks itself; the reference arm runs on rank 0 only and
    reports n_gpus = 2 (the other rank exits 0 without work)."""
    d = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "wan13b_480p"],
             600)
    assert d["impl"] == "reference" and d["n_gpus"] == 2


@pytest.mark.gpu
def test_gpu_arm_two_ranks(tmp_path):
    """--gpus 2 self-launches two ranks (sharing cuda:0 on a 1-GPU box: gloo for the timing collectives),
    heads split 6/6 at C1, max-over-ranks timing; every head's output is bit-identical to the 1-rank run."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    one, two = tmp_path / "n1", tmp_path / "n2"
    d1 = _run(["--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e", "--config", "wan13b_480p",
               "--dump-out", str(one)], 900)
    d2 = _run(["--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e", "--config", "wan13b_480p",
               "--dump-out", str(two)], 900)
    _common(d2)
    assert d1["n_gpus"] == 1 and d2["n_gpus"] == 2
    assert d2["config"]["heads_per_gpu"] == 6
    h1 = json.load(open(one / "rank0.json"))
    h2 = {**json.load(open(two / "rank0.json")), **json.load(open(two / "rank1.json"))}
    assert sorted(h1, key=int) == sorted(h2, key=int) == [str(h) for h in range(12)]
    assert h1 == h2
