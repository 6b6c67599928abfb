"""Multi-process host logic of bench.py on CPU (gloo, world_size 2): the
replica harness's barrier / max-over-ranks / sum-over-ranks helpers, and the
reference arm launched the way the driver launches N>1 runs (torchrun; rank 0
alone prints the JSON line, the other ranks exit 0)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, str(ROOT))
    import bench
    r, w, _ = bench.dist_setup()
    bench.barrier(w)
    mx = bench.allmax(w, float(10 + r))
    sm = bench.allsum(w, float(r + 1))
    import torch.distributed as dist
    dist.destroy_process_group()
    q.put((r, w, mx, sm))


def test_replica_reductions_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out == [(0, 2, 11.0, 3.0), (1, 2, 11.0, 3.0)]


@pytest.mark.timeout(300)
def test_reference_arm_under_torchrun_world2():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
           "--impl", "reference", "--gpus", "2", "--config", "0", "--steps", "3", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=280)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 3
    assert d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
    assert len(d["m_per_step"]) == 3  # the timed steps
