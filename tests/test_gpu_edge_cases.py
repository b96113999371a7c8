"""Edge cases against the reference's own outcomes (tests/golden/make_edge_golden.py):
an empty trace, one request, a relQuery without requests (the reference idles and
aborts), a request using exactly the whole KV budget and one over it, a row longer
than max_num_batched_tokens, a ragged burst with more rows than max_num_seqs, and
all-tied arrivals ordered by rel_id -- every policy, on the device and on the oracle."""

import gzip
import json

import pytest

import edge_cases
from golden_util import GOLDEN_DIR
from paper_2601_11546_b200 import (ArrivalTrace, InfeasibleRequestError, RelQuery, Request, SchedulerConstraints,
                                   SimulationAborted, world_preset)
from paper_2601_11546_b200.engine import EngineConfig, run

with gzip.open(GOLDEN_DIR / "edge" / "edge_cases.json.gz", "rt") as _f:
    GOLD = json.load(_f)
KEYS = sorted(GOLD)
ERRORS = {"SimulationAborted": SimulationAborted, "InfeasibleRequestError": InfeasibleRequestError}


def _case(key):
    name, pol = key.split("/")
    spec = edge_cases.CASES[name]
    trace = edge_cases.build(spec, ArrivalTrace, RelQuery, Request)
    return trace, pol, EngineConfig(constraints=SchedulerConstraints(*spec["constraints"])), GOLD[key]


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_device_edge_case_matches_reference(key):
    trace, pol, cfg, want = _case(key)
    if "raises" in want:
        with pytest.raises(ERRORS[want["raises"]]):
            run(trace, pol, world_preset("opt-13b-like"), cfg)
        return
    r = run(trace, pol, world_preset("opt-13b-like"), cfg)
    assert r.iterations == want["iterations"]
    assert r.sim_duration.hex() == want["clock"]
    assert [[e.iteration, e.case, e.action] for e in r.decision_log] == want["log"]
    got = {str(k): [v.arrival, v.first_prefill_start, v.last_prefill_end, v.last_decode_end]
           for k, v in sorted(r.ledgers.items())}
    assert got == want["ledgers"]


@pytest.mark.parametrize("key", KEYS)
def test_oracle_edge_case_matches_reference(key, oracle_mod):
    """CPU: the checker agrees with the reference on the same cases."""
    trace, pol, cfg, want = _case(key)
    res = oracle_mod.run(trace, pol, world_preset("opt-13b-like"), cfg)
    if "raises" in want:  # the oracle reports the reference's exceptions as status codes
        assert res.status == {"InfeasibleRequestError": 2, "SimulationAborted": 4}[want["raises"]], res.message
        return
    assert res.status == 0, res.message
    assert res.iterations == want["iterations"]
    assert float(res.clock).hex() == want["clock"]
