"""Device unit entry points: PEM batch and the numpy choice replay."""

import numpy as np
import pytest

from paper_2601_11546_b200 import LinearCostModel, SchedulerConstraints, _abi, _native

pytestmark = pytest.mark.gpu

MODEL = LinearCostModel(0.001, 0.02, 0.0002, 0.015)


def test_pem_known_answer():
    c = SchedulerConstraints(cap=1000, max_num_seqs=10, max_num_batched_tokens=500)
    v = _native.pem_batch(np.array([0, 3]), np.array([100, 60, 40]), np.array([2, 2, 2], np.int32),
                          np.zeros(3, np.uint8), c, MODEL)
    assert v[0] == pytest.approx(0.22 + 2 * 0.0156)


@pytest.mark.parametrize("seed", range(6))
def test_pem_batch_matches_oracle(seed, oracle_mod):
    rs = np.random.default_rng(seed)
    cons = [SchedulerConstraints(1000, 10, 200), SchedulerConstraints(150, 10, 150),
            SchedulerConstraints(10_000, 2, 10_000), SchedulerConstraints(200_000, 256, 8192),
            SchedulerConstraints(4000, 16, 512)][seed % 5]
    sets = []
    for _ in range(300):
        n = int(rs.integers(0, 1500 if seed % 2 else 60))
        q = int(rs.integers(0, n + 1))
        pre = np.zeros(n, np.uint8)
        pre[:q] = 1
        utok = rs.integers(0, min(cons.cap, 400) + 1, size=n)
        utok[pre == 1] = 0
        rem = rs.integers(1, 40, size=n).astype(np.int32)
        sets.append((utok, rem, pre))
    off = np.cumsum([0] + [len(s[0]) for s in sets])
    got = _native.pem_batch(off, np.concatenate([s[0] for s in sets]).astype(np.int64),
                            np.concatenate([s[1] for s in sets]).astype(np.int32),
                            np.concatenate([s[2] for s in sets]).astype(np.uint8), cons, MODEL)
    for i, (u, r, p) in enumerate(sets):
        assert got[i] == oracle_mod.pem(u, r, p, cons, MODEL), i


def test_choice_sequence_matches_numpy():
    g = np.random.default_rng(np.random.SeedSequence([3, 0xD9]))
    st = _abi.Pcg64State.from_numpy(g.bit_generator.state)
    rs = np.random.default_rng(0)
    ns = rs.integers(2, 5000, size=500)
    ks = np.minimum(ns - 1, rs.integers(1, 9, size=500))
    got = _native.choice_sequence(st, ns, ks)
    want = np.concatenate([g.choice(int(n), size=int(k), replace=False) for n, k in zip(ns, ks)])
    assert got.tolist() == want.tolist()
    assert st.to_numpy()["state"] == g.bit_generator.state["state"]


def test_waiting_argmin_matches_reference_sort():
    """rs_waiting_argmin == waiting.sort(key=(priority, arrival, rel_id))[0] and len(waiting)
    (engine.py:277-281, 161-176) on entries in admission order, ties included."""
    from paper_2601_11546_b200._native import waiting_argmin

    r = np.random.default_rng(5)
    for n in (0, 1, 7, 512, 513, 5000, 70_000):
        prio = r.choice([0.0, 0.25, 1.5, 3.0, -0.5, -4.0], n) if n % 2 else r.uniform(-10, 10, n)
        wait = r.random(n) < 0.6
        head, count = waiting_argmin(prio, wait)
        ranks = np.flatnonzero(wait)
        assert count == len(ranks)
        if not len(ranks):
            assert head == -1
            continue
        # admission order is (arrival, rel_id), so rank order breaks priority ties
        assert head == ranks[np.lexsort((ranks, prio[ranks]))[0]]
    assert waiting_argmin(np.array([1.0, -2.0]), np.array([1, 1])) == (1, 2)  # sp priorities may be negative
    for bad in (np.nan, -0.0):
        with pytest.raises(ValueError):
            waiting_argmin(np.array([1.0, bad]), np.array([1, 1]))


def test_pem_reference_tests():
    """pkg/tests/test_priority.py TestPem (:180-200) through the drop-in `pem`."""
    from paper_2601_11546_b200 import RemainderItem, pem

    model = LinearCostModel(0.001, 0.02, 0.0002, 0.015)
    c = SchedulerConstraints(cap=1000, max_num_seqs=10, max_num_batched_tokens=500)
    items = [RemainderItem(None, u, 2, False) for u in (100, 60, 40)]
    assert pem(items, c, model) == pytest.approx(0.22 + 2 * 0.0156)
    assert pem([], c, model) == 0.0
    lo = pem([RemainderItem(None, 50, 3, False)] * 4, c, model)
    hi = pem([RemainderItem(None, 100, 3, False)] * 4, c, model)
    assert hi >= lo
    full = pem([RemainderItem(None, 80, 4, False)] * 6, c, model)
    assert pem([RemainderItem(None, 80, 4, False)] * 5, c, model) <= full


@pytest.mark.parametrize("n", [0, 1, 2, 1000, 4096, 4097, 40_000, 65537, 300_000])
def test_radix_sort_is_a_stable_sort(n):
    """North-star kernel 2 (rs_sort_pairs): equals numpy's stable argsort, duplicates
    keeping their input order; keys built like the engine's (okey of priorities of
    either sign, many ties)."""
    rs = np.random.default_rng(n)
    prio = rs.choice(np.concatenate([rs.normal(0, 50, 64), [0.0, 1.5, -2.25]]), size=n)
    keys = _native.priority_keys(prio)
    if n > 2:
        keys[: n // 3] = rs.integers(0, 2**63, size=n // 3, dtype=np.uint64) * np.uint64(2)  # full-width keys too
    vals = np.arange(n, dtype=np.int32)
    ko, vo = _native.sort_pairs(keys, vals)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(vo, vals[order]) and np.array_equal(ko, keys[order])


@pytest.mark.parametrize("n", [3000, 50_000])
def test_radix_sort_equal_and_sorted_keys(n):
    """Every pass the identity (all keys equal), and an already sorted input with ties: the
    grid passes recognise identity passes on the device (radix_sort.cuh)."""
    vals = np.arange(n, dtype=np.int32)
    for keys in (np.full(n, 0x3FF0000000000000, dtype=np.uint64),
                 np.sort(np.random.default_rng(n).integers(0, 1000, n).astype(np.uint64))):
        ko, vo = _native.sort_pairs(keys, vals)
        assert np.array_equal(ko, keys) and np.array_equal(vo, vals)


def test_priority_keys_order_numbers():
    x = np.array([-np.inf, -1e300, -2.5, -1.0, -5e-324, 0.0, 5e-324, 1.0, 2.5, 1e300, np.inf])
    k = _native.priority_keys(x)
    assert np.all(np.diff(k.astype(object)) > 0)
