"""GPU: bench.py's N>1 path end to end under torchrun.

The driver's scaling run launches `bench.py` with one rank per GPU over NCCL;
this box has one GPU, so the same path runs here with two ranks sharing it
over gloo (CBX_BENCH_BACKEND=gloo, ranks mapped onto devices round-robin):
per-rank stream shards, the timing barriers, the max-over-ranks reduction,
rank 0 alone printing one JSON line whose value is the whole-job rate, and
the reference arm (rank 0 alone; other ranks exit 0).
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(args, env_extra, timeout):
    env = dict(os.environ, **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py")] + args
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    return lines


@pytest.mark.gpu
def test_bench_two_ranks_one_json_line():
    lines = _torchrun(["--gpus", "2", "--steps", "3", "--warmup", "3", "--streams", "2", "--no-cpu", "--no-e2e"],
                      {"CBX_BENCH_BACKEND": "gloo"}, timeout=600)
    assert len(lines) == 1, lines  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["value"] > 0 and d["ms_per_step"] > 0
    # whole-job rate: both ranks' streams over the slowest rank's time
    assert abs(d["value"] - 2 * 2 * 3 / (d["ms_per_step"] * 3 / 1000.0)) / d["value"] < 1e-6
    assert d["config"]["parallelism"] == "streams x2"


@pytest.mark.gpu
def test_reference_arm_two_ranks():
    lines = _torchrun(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--ref-budget", "5"],
                      {}, timeout=600)
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0
