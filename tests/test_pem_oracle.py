"""Oracle pem() against the reference's own known answers (pkg/tests/test_priority.py)."""

import pytest

from paper_2601_11546_b200 import LinearCostModel, SchedulerConstraints

MODEL = LinearCostModel(0.001, 0.02, 0.0002, 0.015)


def test_arithmetic_over_decomposition(oracle_mod):
    # test_priority.py:180-186: one prefill batch of 200 uncached tokens, 2 decodes of 3
    c = SchedulerConstraints(cap=1000, max_num_seqs=10, max_num_batched_tokens=500)
    v = oracle_mod.pem([100, 60, 40], [2, 2, 2], [0, 0, 0], c, MODEL)
    assert v == pytest.approx(0.22 + 2 * 0.0156)


def test_empty_is_zero(oracle_mod):
    c = SchedulerConstraints(cap=1000, max_num_seqs=10, max_num_batched_tokens=200)
    assert oracle_mod.pem([], [], [], c, MODEL) == 0.0


def test_infeasible(oracle_mod):
    from paper_2601_11546_b200 import InfeasibleRequestError

    c = SchedulerConstraints(cap=1000, max_num_seqs=10, max_num_batched_tokens=200)
    with pytest.raises(InfeasibleRequestError):
        oracle_mod.pem([2000], [1], [0], c, MODEL)
