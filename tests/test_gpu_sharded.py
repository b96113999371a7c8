"""Sharded pool (BASELINE config 5): relQueries owned round-robin by
admission rank across shards that allgather their heads and priorities every
iteration (csrc/shard.cuh).  On one GPU every shard is a CTA of one launch
exchanging through global memory -- the same device code that runs one shard
per GPU over NVLink peer memory.  Parity bar: bit-identical to the reference
goldens, to the unsharded engine and to the CPU oracle."""

import math

import numpy as np
import pytest

import parity
from golden_util import golden_names, load_golden

pytestmark = pytest.mark.gpu

FIELDS = ("iteration", "clock", "m_plus", "m_minus", "delta_plus", "delta_minus", "delta_total", "kv_reserved",
          "action", "kase", "head", "n_waiting", "batch_rq", "batch_first", "batch_n", "n_reestimated")


def run(trace, policy, world, cfg, pm, seed, shards):
    from paper_2601_11546_b200.engine import Engine, SimulationAborted

    eng = Engine(trace, policy, world, cfg, pm, seed, device=0, shards=shards)
    aborted = None
    try:
        res = eng.run()
    except SimulationAborted as e:
        aborted = str(e)
        res = eng.result
    eng.close()
    return res, aborted


def same_run(a, b):
    assert a.iterations == b.iterations
    assert a.sim_duration == b.sim_duration
    for k in FIELDS:
        assert np.array_equal(a.records[k], b.records[k], equal_nan=a.records[k].dtype.kind == "f"), k
    assert np.array_equal(a.completion_iteration, b.completion_iteration)
    assert (a.cache_hit_tokens, a.cache_miss_tokens) == (b.cache_hit_tokens, b.cache_miss_tokens)


GOLDEN = [n for n in golden_names() if not n.startswith("cfg2") and not n.startswith("cfg3")]


@pytest.mark.parametrize("shards", [2, 3, 8])
@pytest.mark.parametrize("name", GOLDEN)
def test_sharded_matches_reference_golden(name, shards):
    g = load_golden(name)
    trace, policy, world, cfg, pm, seed = parity.golden_inputs(g)
    res, aborted = run(trace, policy, world, cfg, pm, seed, shards)
    assert (aborted is None) == (g["aborted"] is None)
    parity.compare_records(res.records, g, trace, f"sharded{shards}/{name}")
    parity.compare_completion(res.completion_iteration, g, trace)
    assert res.iterations == g["result"]["iterations"]
    assert res.sim_duration == g["result"]["sim_duration"]


@pytest.mark.parametrize("name", ["cfg2_window", "cfg3_window"])
def test_sharded_matches_reference_golden_1m(name):
    """10^6-request windows (configs 2 and 3) over 8 shards."""
    g = load_golden(name)
    trace, policy, world, cfg, pm, seed = parity.golden_inputs(g)
    res, aborted = run(trace, policy, world, cfg, pm, seed, 8)
    assert (aborted is None) == (g["aborted"] is None)
    parity.compare_records(res.records, g, trace, f"sharded8/{name}")


def test_sharded_equals_unsharded_config5_shape(oracle_mod):
    """Config-5 shape scaled down: heavy-tailed outputs, U[1,399] rows, llama-70b-like;
    a window of iterations, sharded 8 ways == unsharded == oracle."""
    from dataclasses import replace

    from paper_2601_11546_b200 import EngineConfig, generate_heavy_tail_trace, world_preset

    trace = generate_heavy_tail_trace(num_relqueries=1500, size_range=(1, 399), rate=1e6, seed=5)
    w = world_preset("llama-70b-like")
    cfg = replace(EngineConfig(), iteration_limit=1500)
    a, ab_a = run(trace, "relserve", w, cfg, None, 0, 1)
    b, ab_b = run(trace, "relserve", w, cfg, None, 0, 8)
    assert ab_a is not None and ab_b is not None  # windowed: the limit ends both
    same_run(a, b)
    ref = oracle_mod.run(trace, "relserve", w, cfg, None, 0)
    n = len(b.records)
    for k in ("clock", "action", "kase", "head", "n_waiting", "batch_rq", "batch_first", "batch_n", "kv_reserved"):
        assert np.array_equal(b.records[k], ref.log[k][:n]), k


@pytest.mark.parametrize("policy,tau", [("relserve-pp", math.inf), ("relserve", 0.05), ("sp", math.inf),
                                        ("fcfs", math.inf)])
def test_sharded_policies(policy, tau, oracle_mod):
    from paper_2601_11546_b200 import EngineConfig, TraceConfig, generate_trace, world_preset

    trace = generate_trace(TraceConfig(num_relqueries=120, size_range=(1, 150), rate=4.0, seed=41))
    w = world_preset("opt-13b-like")
    cfg = EngineConfig(tau=tau, capacity_blocks=400)
    a, _ = run(trace, policy, w, cfg, None, 3, 1)
    b, _ = run(trace, policy, w, cfg, None, 3, 5)
    same_run(a, b)
    ref = oracle_mod.run(trace, policy, w, cfg, None, 3)
    assert ref.status == 0
    assert b.iterations == ref.iterations and b.sim_duration == ref.clock
    assert np.array_equal(b.completion_iteration, ref.completion_iter)


def test_two_process_shards_over_ipc(tmp_path):
    """Two processes, one shard each, mailboxes mapped with CUDA IPC and handles
    swapped over a gloo group (sharded.connect): the multi-GPU code path, here with
    both processes time-sliced on GPU 0.  Bit-identical to the unsharded run."""
    import socket
    import subprocess
    import sys
    from pathlib import Path

    from paper_2601_11546_b200 import EngineConfig, TraceConfig, generate_trace, world_preset

    iters = 30
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    worker = Path(__file__).with_name("ipc_shard_worker.py")
    env = dict(__import__("os").environ, RS_IPC_ITERS=str(iters))
    procs = [subprocess.Popen([sys.executable, str(worker), str(r), "2", str(port), str(tmp_path / f"r{r}.npy")],
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT) for r in range(2)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=240)[0].decode()[-2000:])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    assert all(p.returncode == 0 for p in procs), outs
    trace = generate_trace(TraceConfig(num_relqueries=40, size_range=(1, 60), rate=4.0, seed=9))
    ref, _ = run(trace, "relserve", world_preset("opt-13b-like"), EngineConfig(iteration_limit=iters), None, 0, 1)
    for r in range(2):
        got = np.load(tmp_path / f"r{r}.npy")
        assert len(got) == len(ref.records) == iters
        for k in FIELDS:
            assert np.array_equal(got[k], ref.records[k], equal_nan=got[k].dtype.kind == "f"), (r, k)
