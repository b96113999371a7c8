"""The reference's own arranger tests (pkg/tests/test_arranger.py:100-217),
run through the device arranger (rs_arrange: the engine's arrange() code) --
the Delta worked example, output-limit truncation, scaling with the running
relQueries, and every decision case."""

import math

import numpy as np
import pytest

from paper_2601_11546_b200 import LinearCostModel
from paper_2601_11546_b200._native import arrange

pytestmark = pytest.mark.gpu

MODEL = LinearCostModel(0.001, 0.02, 0.0002, 0.015)  # test_arranger.py:38
PRE, DEC, IDLE = 0, 1, 2  # RS_ACTION_*
PREEMPT, INTERNAL, TRANSITIONAL, FORCED = 0, 1, 2, 3


def proj(running, n_p, utok, ol_p, W, policy="relserve"):
    """project_delta through a transitional decision (m+ < m-, distinct relQueries)."""
    r = arrange(running, d_min_rel_id=running[0][0], prefill_n=n_p, prefill_utok=utok, prefill_rel_id=99,
                prefill_output_limit=ol_p, m_plus=1.0, m_minus=2.0, n_waiting=W, policy=policy, model=MODEL)
    assert r["kase"] == TRANSITIONAL
    return r


def test_worked_example():  # test_arranger.py:102-109
    r = proj([(1, 50)], n_p=20, utok=80, ol_p=50, W=10)
    assert r["delta_plus"] == pytest.approx(0.3)
    assert r["delta_minus"] == pytest.approx(-7.5)
    assert r["delta_total"] == pytest.approx(-7.2)
    assert r["action"] == PRE  # negative Delta prefills


def test_no_waiting_beneficiaries():  # :111-116
    r = proj([(1, 50)], n_p=20, utok=80, ol_p=50, W=0)
    assert r["delta_minus"] == 0.0
    assert r["delta_total"] == r["delta_plus"] > 0


def test_output_limit_truncation_both_ways():  # :118-130
    a = proj([(1, 5)], n_p=10, utok=40, ol_p=100, W=1)
    b = proj([(1, 500)], n_p=10, utok=40, ol_p=100, W=1)
    assert a["delta_plus"] == pytest.approx(MODEL.alpha_p * 40 + MODEL.beta_p + MODEL.alpha_d * 10 * 5)
    assert a["delta_minus"] == pytest.approx(-MODEL.beta_d * 5)
    assert b["delta_minus"] == pytest.approx(-MODEL.beta_d * 100)


def test_scales_with_running_count():  # :132-138
    one = proj([(1, 10)], n_p=10, utok=40, ol_p=10, W=2)
    two = proj([(1, 10), (2, 10)], n_p=10, utok=40, ol_p=10, W=2)
    assert two["delta_plus"] == pytest.approx(2 * one["delta_plus"])


def test_projection_is_evaluated_in_rel_id_order():
    # engine.py:406-408 sorts the running relQueries by rel_id; the fp64 sum is left to right
    run = [(7, 13), (3, 29), (5, 2), (1, 31)]
    r = arrange(run, 7, 9, 123, 99, 17, 1.0, 2.0, 3, "relserve", MODEL)
    lp = MODEL.alpha_p * 123 + MODEL.beta_p
    dp = lp * 4
    for _, ol in sorted(run):
        dp += MODEL.alpha_d * 9 * min(ol, 17)
    assert r["delta_plus"] == dp  # bit for bit: same operations, same order
    assert r["delta_minus"] == -(3 * MODEL.beta_d) * min(17, 31)


def dec(m_plus, m_minus, d_rel=1, p_rel=2, n_d=2, n_p=2, **kw):  # the pair() helper, :141-149
    running = [(d_rel, 10)] if n_d else []
    return arrange(running, d_rel, n_p, 100 * n_p, p_rel, 10, m_plus, m_minus, kw.pop("W", 1),
                   kw.pop("policy", "relserve"), MODEL)


def test_both_empty_idle():  # :153-156
    r = dec(None, None, n_d=0, n_p=0)
    assert r["action"] == IDLE and math.isnan(r["m_plus"]) and math.isnan(r["m_minus"])


def test_only_prefill():  # :158-161
    r = dec(None, 1.0, n_d=0)
    assert r["action"] == PRE and r["kase"] == FORCED


def test_only_decode():  # :163-166
    r = dec(1.0, None, n_p=0)
    assert r["action"] == DEC and r["kase"] == FORCED


def test_preemption():  # :168-170
    r = dec(5.0, 1.0)
    assert r["action"] == PRE and r["kase"] == PREEMPT and math.isnan(r["delta_total"])


def test_internal_same_relquery():  # :172-174
    r = dec(3.0, 3.0, d_rel=7, p_rel=7)
    assert r["action"] == PRE and r["kase"] == INTERNAL


def test_transitional_tie_decodes():  # :186-188: Delta_t == 0 decodes
    # no waiting beneficiaries: Delta_t = Delta+ > 0 decodes; an all-zero model gives Delta_t == 0, which decodes too
    r = arrange([(1, 10)], 1, 2, 200, 2, 10, 1.0, 5.0, 0, "relserve", LinearCostModel(0.001, 0.02, 0.0, 0.0))
    assert r["delta_total"] == r["delta_plus"] > 0 and r["action"] == DEC
    z = arrange([(1, 10)], 1, 2, 0, 2, 10, 1.0, 5.0, 0, "relserve", LinearCostModel(0.0, 0.0, 0.0, 0.0))
    assert z["delta_total"] == 0.0 and z["action"] == DEC  # tie -> decode


def test_force_prefill_only_affects_transitional():  # :190-195
    r = dec(1.0, 5.0, W=0, policy="relserve-pp")
    assert r["action"] == PRE and r["kase"] == TRANSITIONAL and r["delta_total"] > 0
    r2 = dec(5.0, 1.0, policy="relserve-dp")
    assert r2["action"] == PRE and r2["kase"] == PREEMPT


def test_force_decode_in_transitional():  # :197-199
    r = dec(1.0, 5.0, W=100, policy="relserve-dp")
    assert r["delta_total"] < 0 and r["action"] == DEC


def test_equal_minima_distinct_relqueries_transitional():  # :201-203
    r = dec(2.0, 2.0, d_rel=1, p_rel=2)
    assert r["kase"] == TRANSITIONAL


@pytest.mark.parametrize("policy", ["fcfs", "sp"])
def test_prefill_first_policies(policy):  # engine.py:387-395
    assert dec(1.0, 5.0, policy=policy)["action"] == PRE
    assert dec(1.0, None, n_p=0, policy=policy)["action"] == DEC
    r = dec(None, None, n_d=0, n_p=0, policy=policy)
    assert r["action"] == IDLE and r["kase"] == FORCED


def test_decision_always_executable():  # the hypothesis property of :206-217, over a seeded grid
    rs = np.random.default_rng(0)
    for _ in range(300):
        mp, mm = (float(x) for x in rs.uniform(0, 100, 2))
        r = dec(mp, mm, W=int(rs.integers(0, 50)))
        assert r["action"] in (PRE, DEC)
        if r["kase"] == PREEMPT:
            assert mp > mm
