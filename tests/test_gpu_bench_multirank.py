"""bench.py's N > 1 logic (CP groups, CP x DP groups, max-over-ranks timing,
the exchange report, rank-0-only JSON) run under torchrun with all ranks on
the one GPU of this pool, exchanging through gloo (JH_BENCH_TEST_GLOO=1, a
test-only switch: the measured multi-GPU path is NCCL, one GPU per rank)."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("nproc,cp,protocol", [(2, 0, "alltoall"), (4, 2, "alltoall"), (2, 0, "allgather_split")])
def test_bench_multirank_logic(nproc, cp, protocol):
    env = dict(os.environ, JH_BENCH_TEST_GLOO="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", str(nproc), "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-max-len",
           "--no-stack", "--no-e2e", "--cp-sweep-gb", "0", "--cp", str(cp), "--protocol", protocol]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    j = json.loads(lines[0])
    assert j["n_gpus"] == nproc and j["value"] > 0 and j["steps"] == 3
    assert j["config"]["parallelism"] == (f"cp{nproc}" if cp == 0 else f"cp{cp}xdp{nproc // cp}")
    assert "test_mode" in j
    rep = j["cp_exchange"]
    first = "all_to_all" if protocol == "alltoall" else "allgather_split"
    assert {first, "kv_all_gather", "dkv_reduce_scatter", "d_w_all_reduce"} <= set(rep["collectives"])
    assert j["config"]["cp_protocol"] == protocol
    assert rep["exposed_ms_max_over_ranks"] >= 0
