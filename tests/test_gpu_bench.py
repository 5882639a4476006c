"""bench.py's output contract on a small run: one JSON line with the keys the driver reads
(metric, value, unit, timing, roofline, e2e, clocks, gpu_launches, cpu_baseline) and
the reference arm's line.  Small sizes (--reps) keep it to seconds."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("config", ["c3", "c4"])
def test_bench_line_contract(config):
    d = run_bench("--config", config, "--reps", "20", "--steps", "3", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "gpu_launches", "clocks", "e2e", "cpu_baseline"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "alu" and r["peak"] > 0 and r["frac"] > 0
    # a roofline fraction: the timed kernels' own counted work cannot beat the issue peak
    assert r["frac"] <= 1.0 and r["ops_per_step"] / (r["dominant_ms_per_step"] / 1e3) <= r["peak"] * 1e12
    if config == "c3":  # the direct (per-candidate) path, measured in the same run
        dr = r["direct"]
        assert dr["value"] > 0 and 0 < dr["frac"] <= 1.0 and dr["ms_per_launch"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    assert d["config"]["workload"].startswith(config)


def test_bench_reference_arm():
    d = run_bench("--impl", "reference", "--reps", "20", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


@pytest.mark.parametrize("split", ["weak", "sets", "ranks"])
def test_bench_two_ranks(split):
    """The N > 1 launch the driver uses (torchrun, one process per rank, max-over-ranks
    timing), with both ranks sharing the test box's one GPU over gloo: one JSON line from
    rank 0 with n_gpus = 2; graph-mode replay for the set splits, eager for the rank
    windows (whose per-set merge is a host-driven collective)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, GP_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--config", "c3", "--reps", "64", "--split", split,
                          "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-direct"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["scaling"] == ("weak" if split == "weak" else "strong")
    launch = d["config"]["launch"]
    assert launch.startswith("CUDA graphs") if split != "ranks" else launch == "eager"
