"""Device engine parity: bit-exact against the real reference's golden runs and
against the CPU oracle on further seeded traces."""

import math

import numpy as np
import pytest

import parity
from golden_util import golden_names, load_golden

pytestmark = pytest.mark.gpu


def run_device(trace, policy, world, cfg, pm, seed):
    from paper_2601_11546_b200.engine import Engine, SimulationAborted

    eng = Engine(trace, policy, world, cfg, pm, seed, device=0)
    aborted = None
    try:
        res = eng.run()
    except SimulationAborted as e:
        aborted = str(e)
        res = eng.result
    eng.close()
    return res, aborted


@pytest.mark.parametrize("name", golden_names())
def test_device_matches_reference_golden(name):
    g = load_golden(name)
    trace, policy, world, cfg, pm, seed = parity.golden_inputs(g)
    res, aborted = run_device(trace, policy, world, cfg, pm, seed)
    assert (aborted is None) == (g["aborted"] is None)
    parity.compare_records(res.records, g, trace, f"device/{name}")
    parity.compare_completion(res.completion_iteration, g, trace)
    led = res.ledgers
    c = trace.columns()
    fps = np.array([led[int(r)].first_prefill_start if int(r) in led and led[int(r)].first_prefill_start is not None
                    else math.nan for r in c.rel_id])
    lpe = np.array([led[int(r)].last_prefill_end if int(r) in led and led[int(r)].last_prefill_end is not None
                    else math.nan for r in c.rel_id])
    lde = np.array([led[int(r)].last_decode_end if int(r) in led and led[int(r)].last_decode_end is not None
                    else math.nan for r in c.rel_id])
    parity.compare_ledgers(fps, lpe, lde, g, trace)
    want = g["result"]
    assert res.iterations == want["iterations"]
    assert res.sim_duration == want["sim_duration"]
    assert res.cache_hit_tokens == want["cache_hit_tokens"]
    assert res.cache_miss_tokens == want["cache_miss_tokens"]
    assert len(res.ledgers) == len(g["ledgers"])


CASES = [
    # (trace config, policy, world, engine config kwargs, seed)
    (dict(num_relqueries=60, size_range=(1, 200), rate=2.0, seed=31), "relserve", "opt-13b-like", {}, 1),
    (dict(num_relqueries=40, size_range=(50, 300), rate=50.0, seed=32), "relserve", "llama-70b-like",
     dict(capacity_blocks=300), 2),
    (dict(num_relqueries=50, size_range=(1, 80), rate=3.0, seed=33), "relserve-pp", "qwen-32b-like",
     dict(tau=0.2), 3),
    (dict(num_relqueries=50, size_range=(1, 80), rate=3.0, seed=34), "relserve-dp", "opt-13b-like",
     dict(sample_size=5, capacity_blocks=150), 4),
    (dict(num_relqueries=30, size_range=(1, 120), rate=1.0, seed=35, mean_input_len=64), "relserve",
     "opt-13b-like", dict(block_size=8, capacity_blocks=90), 5),
    (dict(num_relqueries=80, size_range=(1, 40), rate=10.0, seed=36), "sp", "opt-13b-like", {}, 0),
    (dict(num_relqueries=80, size_range=(1, 40), rate=10.0, seed=37), "fcfs", "llama-70b-like",
     dict(capacity_blocks=200), 0),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_device_matches_oracle_random_traces(case, oracle_mod):
    from paper_2601_11546_b200 import EngineConfig, SchedulerConstraints, TraceConfig, generate_trace, world_preset

    tc, policy, world, kw, seed = CASES[case]
    trace = generate_trace(TraceConfig(**tc))
    cfg = EngineConfig(**kw)
    w = world_preset(world)
    ref = oracle_mod.run(trace, policy, w, cfg, None, seed)
    assert ref.status == 0, ref.message
    res, aborted = run_device(trace, policy, w, cfg, None, seed)
    assert aborted is None
    assert res.iterations == ref.iterations
    for k in ref.log.dtype.names:
        a, b = res.records[k], ref.log[k]
        if a.dtype.kind == "f":
            assert np.array_equal(a, b, equal_nan=True), k
        else:
            assert np.array_equal(a, b), k
    assert np.array_equal(res.completion_iteration, ref.completion_iter)
    assert res.sim_duration == ref.clock
    assert (res.cache_hit_tokens, res.cache_miss_tokens) == (ref.cache_hit_tokens, ref.cache_miss_tokens)


@pytest.mark.parametrize("chunk", [3, 64])
def test_noise_prefix_refill_matches_reference_golden(chunk, monkeypatch):
    """World-model noise handed to the device in short prefixes (launches stop when
    they run out, the host doubles the prefix) gives the reference's run."""
    from paper_2601_11546_b200.engine import Engine

    monkeypatch.setattr(Engine, "noise_chunk", chunk)
    g = load_golden("noise_relserve")
    trace, policy, world, cfg, pm, seed = parity.golden_inputs(g)
    res, aborted = run_device(trace, policy, world, cfg, pm, seed)
    assert aborted is None
    parity.compare_records(res.records, g, trace, f"noise/{chunk}")
    parity.compare_completion(res.completion_iteration, g, trace)
    assert res.sim_duration == g["result"]["sim_duration"]


@pytest.mark.parametrize("name", golden_names())
def test_device_parity_mode_matches_reference(name):
    """Parity mode on every golden: the priority update of every iteration (each live
    relQuery's value, reused and override flags, priority.py:287-315, and the DPU generator
    state after it) and -- where the golden recorded it -- the whole waiting queue
    (engine.py:277-281, sorted by (priority, arrival, rel_id); rebuilt from the priorities by
    the device radix sort) equal the reference's, bit for bit, along with every decision."""
    from paper_2601_11546_b200.engine import Engine, SimulationAborted

    g = load_golden(name)
    trace, policy, world, cfg, pm, seed = parity.golden_inputs(g)
    eng = Engine(trace, policy, world, cfg, pm, seed, device=0, record_waiting_order=True)
    try:
        res = eng.run()
    except SimulationAborted:
        res = eng.result
    eng.close()
    parity.compare_records(res.records, g, trace, f"parity/{name}")
    rel = trace.columns().rel_id
    n = 0
    for e in g["iters"]:
        if "order" in e:
            got = [int(rel[i]) for i in res.waiting_orders[e["it"]]]
            assert got == e["order"], f"{name}: waiting order differs at iteration {e['it']}"
            n += 1
        assert len(res.waiting_orders[e["it"]]) == e["W"]
    if policy in ("fcfs", "sp"):
        assert res.priority_records is None
    else:
        assert parity.compare_priority_records(res, g, name) == len(g["iters"])


def test_pinned_trace_and_result_readback():
    """Page-locked trace columns (the e2e path) give the identical run; the int32
    completion readback equals read_requests' completion column; the lazily built
    ledgers / sizes equal an eager build."""
    from paper_2601_11546_b200 import EngineConfig, TraceConfig, generate_trace, world_preset
    from paper_2601_11546_b200.engine import Engine

    tc = TraceConfig(num_relqueries=60, size_range=(1, 90), rate=6.0, seed=17)
    w = world_preset("opt-13b-like")
    a, _ = run_device(generate_trace(tc), "relserve", w, EngineConfig(), None, 3)
    pinned = generate_trace(tc).pin_memory()
    assert all(getattr(pinned.columns(), f).flags["C_CONTIGUOUS"] for f in ("tok", "out", "row_off"))
    eng = Engine(pinned, "relserve", w, EngineConfig(), None, 3, device=0)
    b = eng.run()
    _, _, comp64, _ = eng.requests_state
    eng.close()
    assert b.completion_iteration.dtype == np.int32
    assert np.array_equal(b.completion_iteration, comp64)
    assert np.array_equal(a.completion_iteration, b.completion_iteration)
    for k in a.records.dtype.names:
        assert np.array_equal(a.records[k], b.records[k], equal_nan=a.records[k].dtype.kind == "f"), k
    assert dict(a.ledgers) == dict(b.ledgers) and len(b.ledgers) == 60
    c = pinned.columns()
    assert dict(b.relquery_sizes) == {int(r): int(s) for r, s in zip(c.rel_id, np.diff(c.row_off))}


@pytest.mark.parametrize("big", [False, True])
@pytest.mark.parametrize("ident", [True, False])
def test_creation_row_checks(ident, big):
    """engine.py:235-239 and the device model's row limits, checked on the device
    (admission order == trace order, >= 2^16 rows) or on the host (otherwise): same
    exception, same message naming the offending request."""
    from paper_2601_11546_b200 import EngineConfig, SchedulerConstraints, world_preset
    from paper_2601_11546_b200.engine import Engine
    from paper_2601_11546_b200.priority import InfeasibleRequestError
    from paper_2601_11546_b200.workload import ArrivalTrace, TraceColumns

    n0, n1 = (40_000, 40_000) if big else (2, 3)

    def trace(bad_tok=None, bad_out=None):
        tok = np.full(n0 + n1, 100, np.int32)
        out = np.full(n0 + n1, 5, np.int32)
        if bad_tok is not None:
            tok[n0 + 1] = bad_tok
        if bad_out is not None:
            out[n0 + 1] = bad_out
        ids = [3, 7] if ident else [7, 3]  # equal arrivals: admission order is by rel_id
        return ArrivalTrace(columns=TraceColumns(
            rel_id=np.array(ids, np.int64), arrival=np.zeros(2), output_limit=np.array([10, 10], np.int32),
            prefix_len=np.zeros(2, np.int32), row_off=np.array([0, n0, n0 + n1], np.int64),
            tok=tok, out=out, token_seed=0))

    w = world_preset("opt-13b-like")
    cfg = EngineConfig(constraints=SchedulerConstraints(cap=500, max_num_seqs=16, max_num_batched_tokens=400),
                       iteration_limit=50)
    Engine(trace(), "relserve", w, cfg, None, 0, device=0).close()
    with pytest.raises(ValueError, match="non-empty"):
        Engine(trace(bad_tok=0), "relserve", w, cfg, None, 0, device=0)
    with pytest.raises(ValueError, match="out of range"):
        Engine(trace(bad_out=11), "relserve", w, cfg, None, 0, device=0)
    rid = 7 if ident else 3  # the second relQuery in trace order
    with pytest.raises(InfeasibleRequestError, match=rf"request {rid}/1 needs 501 KV tokens > cap 500"):
        Engine(trace(bad_tok=491), "relserve", w, cfg, None, 0, device=0)
