"""DynamicPriorityUpdater (priority.py:238-339) as a library API: the device-backed
updater equals relsim's record for record -- values bit-identical, reuse and
starvation flags, iteration_computed, and the generator state after every update
-- over the scripted update sequences of tests/dpu_scenario.py
(goldens: tests/golden/make_dpu_golden.py)."""

import gzip
import json

import numpy as np
import pytest

import dpu_scenario
from golden_util import GOLDEN_DIR
from paper_2601_11546_b200 import (DynamicPriorityUpdater, LinearCostModel, RelQuery, Request,
                                   SchedulerConstraints, priority, utok_approx)


def _golden(name):
    with gzip.open(GOLDEN_DIR / "dpu_api" / f"{name}.json.gz", "rt") as f:
        return json.load(f)


def _replay(name):
    g = _golden(name)
    seed, n_rq, iters, tau, k = dpu_scenario.SCENARIOS[name]
    rqs = dpu_scenario.build(seed, n_rq, Request, RelQuery)
    cache = dpu_scenario.StubCache()
    dpu = DynamicPriorityUpdater(SchedulerConstraints(*g["constraints"]), LinearCostModel(*g["model"]), cache,
                                 sample_size=k, tau=tau,
                                 rng=np.random.default_rng(np.random.SeedSequence([seed, 0xD9])))
    recs, states = dpu_scenario.drive(dpu, cache, rqs, iters, seed)
    return g, recs, states


def _check(g, recs, states):
    assert len(recs) == len(g["records"])
    for it, (got, want) in enumerate(zip(recs, g["records"])):
        assert [(r, v.hex(), ic, ru, ov) for r, v, ic, ru, ov in got] == [tuple(w) for w in want], it
    assert [(str(s), h, u) for s, h, u in states] == [tuple(w) for w in g["rng"]]


@pytest.mark.parametrize("name", sorted(dpu_scenario.SCENARIOS))
def test_updater_host_logic_against_reference(name, oracle_mod, monkeypatch):
    """CPU: reuse rule, sampling, utok*, overrides and RNG stream, with the PEM
    evaluated by the oracle's restatement in place of the device launch."""

    def oracle_pem_batch(rems, cons, model, device=0):
        return np.array([oracle_mod.pem(u, r, p, cons, model) for u, r, p in rems])

    monkeypatch.setattr(priority, "pem_batch", oracle_pem_batch)
    _check(*_replay(name))


def test_utok_approx_known_answers():
    """test_prefix_cache.py:168-187: 200 x 0.38 -> 76, 215 x 0.5 -> 108 (half up)."""
    r1 = Request(0, 0, list(range(200)), 10, 5)
    r2 = Request(0, 1, list(range(215)), 10, 5)
    assert utok_approx(r1, 0.38) == 76
    assert utok_approx(r2, 0.5) == 108
    with pytest.raises(ValueError):
        utok_approx(r1, 1.5)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(dpu_scenario.SCENARIOS))
def test_updater_on_device_matches_reference(name):
    """GPU: every estimate of an update priced by one rs_pem_batch launch."""
    _check(*_replay(name))
