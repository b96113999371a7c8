"""Complete runs at BASELINE's full sizes (configs 2 and 3: 10^6 requests, 206k
and 131k iterations; config 5: 8*10^6 requests sharded 8 ways), checked through
size-independent properties -- what must hold of any correct run to completion:

* every request is prefilled once and decoded to its EOS point: the prefill
  batches of a relQuery cover its rows exactly once, decode batches add up to
  sum(out) row-iterations, every request has a completion iteration;
* token conservation: cache hit + miss tokens == sum(tok) (test_engine.py:197-206);
* batch invariants: kv_reserved <= cap and back to 0, batch sizes <= mns
  (test_engine.py:181-195); the clock never decreases and ends at the last decode;
* ledgers: arrival <= first prefill <= last prefill <= last decode, and the latency
  breakdown sums exactly (test_engine.py:78-88);
* config 5: the 8-shard run equals the unsharded run record for record.

Configs 2 and 3 under every policy are also compared bit for bit with the CPU oracle's complete runs
(about two minutes each on one core; the Python reference would need hours)
through fingerprints: SHA-256 per decision-record field and of the per-request
completion iterations, exact final clock and cache counters
(tests/golden/fullscale.json, made by tests/golden/make_fullscale.py).  The
config-5 pool (≈ 80 oracle iterations/s) is compared with the oracle over its
first 3,000 iterations at full size (first sight of all 40,000 relQueries
included), unsharded and sharded 8 ways; its complete run is checked against the
unsharded device run.
"""

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _trace(config):
    from paper_2601_11546_b200 import (EngineConfig, TraceConfig, generate_heavy_tail_trace, generate_trace,
                                       world_preset)

    if config == 2:
        t = generate_trace(TraceConfig(num_relqueries=1000, size_range=(1000, 1000), rate=1e6, seed=0))
        return t, world_preset("opt-13b-like"), EngineConfig()
    n = 5000 if config == 3 else 40_000
    t = generate_heavy_tail_trace(num_relqueries=n, size_range=(1, 399), rate=1e6, seed=0)
    return t, world_preset("llama-70b-like"), EngineConfig()


def _run(trace, world, cfg, shards=1, policy="relserve"):
    from paper_2601_11546_b200.engine import Engine

    eng = Engine(trace, policy, world, cfg, None, 0, device=0, shards=shards)
    eng.chunk_iterations = 1 << 16
    try:
        res = eng.run()
    finally:
        eng.close()
    return res


def _check_run(res, trace, cfg):
    from paper_2601_11546_b200.report import decompose

    c = trace.columns()
    recs = res.records
    cons = cfg.constraints
    assert len(recs) == res.iterations
    assert np.array_equal(recs["iteration"], np.arange(res.iterations))
    # every request prefilled exactly once, relQuery by relQuery, in row order
    pre = recs[recs["action"] == 0]
    sizes = np.diff(c.row_off)
    order = np.lexsort((c.rel_id, c.arrival))  # admission rank -> trace index
    covered = np.zeros(len(sizes), np.int64)
    np.add.at(covered, order[pre["batch_rq"]], pre["batch_n"])
    assert np.array_equal(covered, sizes)
    # decode batches: one token per running row per decode = sum of EOS points
    dec = recs[recs["action"] == 1]
    assert int(dec["batch_n"].astype(np.int64).sum()) == int(c.out.astype(np.int64).sum())
    assert (res.completion_iteration >= 0).all()
    assert int(res.completion_iteration.max()) == res.iterations - 1
    # conservation and batch invariants
    assert res.cache_hit_tokens + res.cache_miss_tokens == int(c.tok.astype(np.int64).sum())
    assert (recs["kv_reserved"] <= cons.cap).all() and recs["kv_reserved"][-1] == 0
    assert (recs["batch_n"] <= cons.max_num_seqs).all()
    assert (pre["batch_n"] >= 1).all()
    assert (np.diff(recs["clock"]) >= 0).all()
    # ledgers
    assert len(res.ledgers) == len(sizes)
    last = 0.0
    for rel_id, led in res.ledgers.items():
        assert led.complete
        assert led.arrival <= led.first_prefill_start <= led.last_prefill_end <= led.last_decode_end
        b = decompose(rel_id, led)
        assert b.waiting_s + b.core_s + b.tail_s == b.total_s
        last = max(last, led.last_decode_end)
    assert res.sim_duration == last


_FULL = json.loads((Path(__file__).parent / "golden" / "fullscale.json").read_text())
_GOLDEN = _FULL["configs"]
_WINDOWS = _FULL.get("windows", {})


@pytest.mark.parametrize("name", sorted(_GOLDEN))
def test_full_run_properties_and_oracle_fingerprint(name):
    from fullscale_util import RUNS, WORKLOADS, fingerprint

    wl, policy = RUNS[name]
    trace, world, cfg = WORKLOADS[wl]()
    res = _run(trace, world, cfg, policy=policy)
    _check_run(res, trace, cfg)
    g = _GOLDEN[name]
    assert res.iterations == g["iterations"]
    assert repr(float(res.sim_duration)) == g["clock"]
    assert (res.cache_hit_tokens, res.cache_miss_tokens) == (g["cache_hit_tokens"], g["cache_miss_tokens"])
    fp = fingerprint(res.records, res.completion_iteration)
    for k, v in fp.items():
        assert v == g[k], k


def test_config5_sharded_full_run_equals_unsharded():
    trace, world, cfg = _trace(5)
    a = _run(trace, world, cfg, shards=1)
    b = _run(trace, world, cfg, shards=8)
    assert (a.iterations, a.sim_duration) == (b.iterations, b.sim_duration)
    for k in a.records.dtype.names:
        assert np.array_equal(a.records[k], b.records[k], equal_nan=a.records[k].dtype.kind == "f"), k
    assert np.array_equal(a.completion_iteration, b.completion_iteration)
    assert (a.cache_hit_tokens, a.cache_miss_tokens) == (b.cache_hit_tokens, b.cache_miss_tokens)
    _check_run(b, trace, cfg)


@pytest.mark.parametrize("shards", [1, 8])
@pytest.mark.parametrize("name", sorted(_WINDOWS))
def test_full_size_window_equals_oracle(name, shards):
    """Config 5 at full size (8e6 requests in one pool), the first 3,000 iterations: the
    device run -- unsharded, and sharded 8 ways with the per-iteration exchange -- equals the
    oracle's, record for record (SHA-256 per decision field, per-request completion
    iterations), with the same clock, cache counters and kv at the window's end."""
    from dataclasses import replace

    from fullscale_util import WINDOWS, WORKLOADS, fingerprint
    from paper_2601_11546_b200.engine import Engine, SimulationAborted

    wl, policy, n = WINDOWS[name]
    trace, world, cfg = WORKLOADS[wl]()
    eng = Engine(trace, policy, world, replace(cfg, iteration_limit=n), None, 0, device=0, shards=shards)
    with pytest.raises(SimulationAborted):
        eng.run()
    res = eng.result
    st = eng._status
    eng.close()
    g = _WINDOWS[name]
    assert res.iterations == g["iterations"] == n
    assert repr(float(res.sim_duration)) == g["clock"]
    assert (res.cache_hit_tokens, res.cache_miss_tokens) == (g["cache_hit_tokens"], g["cache_miss_tokens"])
    assert int(st.kv_reserved) == g["kv_reserved"]
    fp = fingerprint(res.records, res.completion_iteration.astype(np.int64))
    for k, v in fp.items():
        assert v == g[k], k
