"""Multi-GPU and multi-rank paths.

* The sharded pool with one process per device: each rank's mailbox is mapped
  into the others with CUDA IPC and the per-iteration exchange runs over NVLink
  peer memory (csrc/shard.cuh) -- skipped unless at least two GPUs are visible
  (every gpurun box has one; the driver's 8-GPU run has eight).
* `bench.py` under torchrun, as the driver launches it: config 2 (independent
  traces, weak scaling) and config 5 (one pool sharded over the ranks) on N
  GPUs when present, and the same multi-rank code paths with two ranks sharing
  GPU 0 (barriers, max-over-ranks timing, the IPC handle exchange) everywhere.
"""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gpus() -> int:
    import torch

    return torch.cuda.device_count()


@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs (one shard per device over NVLink)")
def test_shards_one_per_gpu_equal_unsharded(tmp_path):
    from paper_2601_11546_b200 import EngineConfig, TraceConfig, generate_trace, world_preset
    from paper_2601_11546_b200.engine import Engine, SimulationAborted

    world = min(_gpus(), 4)
    iters = 200
    port = _port()
    env = dict(os.environ, RS_IPC_ITERS=str(iters), RS_IPC_DEVICE_PER_RANK="1", RS_IPC_RELQUERIES="80")
    worker = Path(__file__).with_name("ipc_shard_worker.py")
    procs = [subprocess.Popen([sys.executable, str(worker), str(r), str(world), str(port),
                               str(tmp_path / f"r{r}.npy")], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT) for r in range(world)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=300)[0].decode()[-2000:])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    assert all(p.returncode == 0 for p in procs), outs
    trace = generate_trace(TraceConfig(num_relqueries=80, size_range=(1, 60), rate=4.0, seed=9))
    eng = Engine(trace, "relserve", world_preset("opt-13b-like"), EngineConfig(iteration_limit=iters), device=0)
    with pytest.raises(SimulationAborted):
        eng.run()
    ref = eng.result.records
    eng.close()
    for r in range(world):
        got = np.load(tmp_path / f"r{r}.npy")
        assert len(got) == len(ref) == iters
        for k in ref.dtype.names:
            assert np.array_equal(got[k], ref[k], equal_nan=got[k].dtype.kind == "f"), (r, k)


def _torchrun(n, *args, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"), "--gpus", str(n),
           *args]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def _check_line(d, n):
    assert d["n_gpus"] == n and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 3
    assert d["ms_per_step"] > 0 and d["gpu_launches"] >= 2


@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("config", ["2", "5"])
def test_bench_torchrun_on_gpus(config):
    n = min(_gpus(), 8)
    d = _torchrun(n, "--config", config, "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-e2e")
    _check_line(d, n)
    assert d["scaling"] == ("weak" if config == "2" else "strong")


@pytest.mark.parametrize("config", ["2", "5"])
def test_bench_torchrun_two_ranks_one_gpu(config):
    """The driver's torchrun launch with two ranks sharing GPU 0 (gloo plumbing): one JSON line
    from rank 0, iterations of both ranks' traces (config 2) or of the one sharded pool (config 5,
    mailboxes exchanged over CUDA IPC)."""
    env = dict(os.environ, RS_BENCH_DEVICE="0")
    d = _torchrun(2, "--config", config, "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-e2e",
                  "--iters-per-step", "50", env=env)
    _check_line(d, 2)
    assert d["iterations_timed"] == (2 if config == "2" else 1) * 2 * 50
