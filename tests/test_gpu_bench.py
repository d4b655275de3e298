"""The bench contract end to end on a real GPU: the N = 1 JSON line (C1 size) and the N > 1 path
(two ranks on one GPU over gloo: partitioning, barriers, all-reduce of Z, max-over-ranks timing)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "clocks", "e2e", "gpu_launches", "roofline", "cpu_baseline"}


def _last_json(out):
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


def test_bench_line_n1():
    out = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--steps", "3", "--warmup", "3", "--no-cpu"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = _last_json(out.stdout)
    assert KEYS <= set(line)
    assert line["n_gpus"] == 1 and line["gpu_launches"] > 0 and line["value"] > 0
    assert line["roofline"]["bound"] == "hbm" and 0 < line["roofline"]["frac"] < 2


def test_bench_two_ranks_gloo_one_gpu():
    env = dict(os.environ, CSK_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29671", "bench.py", "--gpus", "2", "--config", "c1", "--steps", "3",
           "--warmup", "3", "--no-cpu", "--no-e2e"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = _last_json(out.stdout)
    assert line["n_gpus"] == 2 and line["config"]["d_global"] == 2 * line["config"]["d_per_rank"]
    assert line["accuracy"]["rel_residual_ms"] < 1.0
