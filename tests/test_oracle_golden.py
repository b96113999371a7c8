"""The CPU oracle reproduces the real reference (golden runs) bit for bit."""

import numpy as np
import pytest

import parity
from golden_util import golden_names, load_golden

NAMES = golden_names()


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_golden(name, oracle_mod):
    O = oracle_mod
    g = load_golden(name)
    trace, policy, world, cfg, pm, seed = parity.golden_inputs(g)
    res = O.run(trace, policy, world, cfg, pm, seed, record=O.OR_REC_DPU | O.OR_REC_WAITING | O.OR_REC_RNG)
    parity.compare_records(res.log, g, trace, f"oracle/{name}")
    parity.compare_completion(res.completion_iter, g, trace)
    parity.compare_ledgers(res.first_prefill_start, res.last_prefill_end, res.last_decode_end, g, trace)
    want = g["result"]
    assert res.iterations == want["iterations"]
    assert res.clock == want["sim_duration"]
    assert res.cache_hit_tokens == want["cache_hit_tokens"]
    assert res.cache_miss_tokens == want["cache_miss_tokens"]
    assert res.kv_reserved == want["kv_reserved"]
    assert res.status == (0 if g["aborted"] is None else 3)
    rel = trace.columns().rel_id
    for it, want_dpu in parity.golden_dpu_by_iter(g).items():
        lo, hi = res.dpu_off[it], res.dpu_off[it + 1]
        got = {int(rel[d["rq"]]): float(d["value"]) for d in res.dpu[lo:hi] if not d["reused"]}
        assert got == want_dpu, f"DPU values differ at iteration {it}"
    for e in g["iters"]:
        if "order" in e:
            lo, hi = res.wait_off[e["it"]], res.wait_off[e["it"] + 1]
            assert [int(rel[i]) for i in res.wait[lo:hi]] == e["order"], f"waiting order it {e['it']}"
        if "rng" in e:  # the DPU generator after update() (numpy bit_generator.state)
            hi, lo, has, u = (int(x) for x in res.rng_trace[e["it"]])
            assert [str((hi << 64) | lo), has, u] == e["rng"], f"DPU RNG state differs at iteration {e['it']}"
    if policy not in ("fcfs", "sp"):
        assert any("rng" in e for e in g["iters"])


def test_goldens_cover_the_scope():
    names = set(NAMES)
    # every policy, windowed 1e6-row configs, eviction pressure, starvation
    for must in ("cfg1_relserve", "cfg1_fcfs", "cfg1_sp", "cfg1_pp", "cfg1_dp", "cfg2_window",
                 "cfg3_window", "evict_tiny", "tau_relserve", "starve_tau"):
        assert must in names
