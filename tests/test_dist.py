"""bench.py's N>1 plumbing (replicas only) on CPU with gloo,
world_size 2: barrier + max-over-ranks timing and the rank-0-only output."""

from __future__ import annotations

import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import os, sys
sys.path.insert(0, os.environ["ROOT"])
import torch.distributed as dist
import bench
dist.init_process_group("gloo", rank=int(os.environ["RANK"]), world_size=int(os.environ["WORLD_SIZE"]))
ws, rank, _ = bench.dist_env()
bench.dist_barrier(ws)
m = bench.dist_max(float(rank + 1) * 1.5, ws)
assert m == 1.5 * ws, m
print("rank", rank, "max", m, flush=True)
dist.destroy_process_group()
"""


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_dist_max_over_two_gloo_ranks():
    port = _free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, ROOT=ROOT, RANK=str(rank), WORLD_SIZE="2", LOCAL_RANK=str(rank),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", CHILD], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=120) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
    assert "max 3.0" in outs[0][0] and "max 3.0" in outs[1][0]


def test_reference_arm_rank_nonzero_exits_quietly():
    """--impl reference under torchrun: ranks != 0 exit 0 without output."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.mark.slow
def test_reference_arm_prints_contract_line():
    import json

    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "impl", "cpu_baseline", "e2e", "higher_is_better"):
        assert k in line
    # the real reference (baseline/_ref) when installed, else the oracle port
    from tools import refcpu

    want = "reference" if refcpu.reference_dir() else "port"
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == want
    assert line["config"]["workload"] == __import__("bench").WORKLOAD
    assert line["cpu_baseline"]["extrapolated"] is True and line["cpu_baseline"]["measured_elements"] > 0
