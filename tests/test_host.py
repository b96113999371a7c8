"""Host-side logic (no GPU): trace generation and files, prefix-structure
marshalling, static priorities, API validation and the no-fallback rule."""

import math

import numpy as np
import pytest

from paper_2601_11546_b200 import (ArrivalTrace, EngineConfig, RelQuery, Request, TraceConfig,
                                   generate_heavy_tail_trace, generate_trace, load_trace, save_trace,
                                   static_relquery_prio, world_preset)
from paper_2601_11546_b200 import _marshal
from paper_2601_11546_b200.engine import Engine, SimulationAborted
from golden_util import digest_columns, digest_entries


def test_v1_round_trip_is_identical(tmp_path):
    t = generate_trace(TraceConfig(num_relqueries=20, size_range=(1, 30), rate=2.0, seed=5))
    p = tmp_path / "t.jsonl"
    save_trace(t, p)
    t2 = load_trace(p)
    assert digest_columns(t.columns()) == digest_columns(t2.columns())
    save_trace(t2, tmp_path / "t2.jsonl")
    assert p.read_bytes() == (tmp_path / "t2.jsonl").read_bytes()


def test_lazy_tokens_follow_the_count_keyed_streams():
    t = generate_trace(TraceConfig(num_relqueries=3, size_range=(4, 4), rate=1.0, seed=2))
    for q in t.entries:
        toks = [r.tokens for r in q.requests]
        assert all(len(x) == r.tok for x, r in zip(toks, q.requests))
        pre = toks[0][: q.prefix_len]
        assert all(x[: q.prefix_len] == pre for x in toks)  # shared prefix
        # the first suffix tokens differ between rows (private tails)
        assert len({tuple(x[q.prefix_len:q.prefix_len + 4]) for x in toks}) == len(toks)
    # entries built from columns and columns rebuilt from entries agree
    assert digest_entries(t.entries) == digest_columns(t.columns())


def test_heavy_tail_trace_is_deterministic_and_bounded():
    a = generate_heavy_tail_trace(num_relqueries=300, seed=4)
    b = generate_heavy_tail_trace(num_relqueries=300, seed=4)
    assert digest_columns(a.columns()) == digest_columns(b.columns())
    ol = a.columns().output_limit
    assert ol.min() >= 8 and ol.max() <= 2048 and (ol > 100).any()


def _rq(rel_id, rows, limit=5, arrival=0.0):
    return RelQuery(rel_id, [Request(rel_id, i, toks, limit, limit, arrival) for i, toks in enumerate(rows)],
                    limit, arrival)


def test_chain_blocks_from_explicit_tokens():
    shared = list(range(100, 132))  # two whole blocks shared by every row
    rows = [shared + [1000 * i + j for j in range(20)] for i in range(1, 4)]
    t = ArrivalTrace([_rq(0, rows)], 1.0, 0)
    m = _marshal.marshal_trace(t, 16, "relserve", world_preset("opt-13b-like"))
    assert m.arrays["chain_blocks"].tolist() == [2]


def test_non_forest_prefix_structure_is_rejected():
    shared = list(range(64))
    a = _rq(0, [shared + [1, 2, 3], shared + [4, 5, 6]])
    b = _rq(1, [shared + [7, 8, 9]])  # shares blocks with relQuery 0
    t = ArrivalTrace([a, b], 1.0, 0)
    with pytest.raises(NotImplementedError):
        _marshal.marshal_trace(t, 16, "relserve", world_preset("opt-13b-like"))


def test_static_priorities_match_python_sum():
    t = generate_trace(TraceConfig(num_relqueries=25, size_range=(1, 60), rate=3.0, seed=9))
    m = world_preset("qwen-32b-like")
    got = _marshal._static_priorities(t, m, None)
    for q, g in zip(t.entries, got):
        want = static_relquery_prio(q, lambda tok: m.alpha_p * tok, lambda ol: m.alpha_d * ol)
        assert g == want  # bit-exact, incl. CPython 3.12's compensated sum


def test_api_validation_before_any_device_work():
    t = generate_trace(TraceConfig(num_relqueries=2, size_range=(1, 3), seed=1))
    w = world_preset("opt-13b-like")
    with pytest.raises(ValueError):
        Engine(t, "srpt", w)
    with pytest.raises(ValueError):
        Engine(t, "relserve", w, EngineConfig(tau=0.0))
    with pytest.raises(ValueError):
        Engine(t, "relserve", w, EngineConfig(noise_sigma=-0.1))


def test_no_cpu_fallback_without_a_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    t = generate_trace(TraceConfig(num_relqueries=2, size_range=(1, 3), seed=1))
    with pytest.raises(RuntimeError):
        Engine(t, "relserve", world_preset("opt-13b-like"))


def test_native_v1_reader_equals_json_reader(tmp_path):
    """csrc/trace_v1.cpp reads exactly what the json-module reader does (workload.py:349-384)."""
    import numpy as np

    from paper_2601_11546_b200 import generate_heavy_tail_trace, load_trace, save_trace
    from paper_2601_11546_b200.workload import load_trace_json

    for i, tr in enumerate([generate_trace(TraceConfig(num_relqueries=50, size_range=(1, 40), rate=2.5, seed=5)),
                            generate_heavy_tail_trace(num_relqueries=200, size_range=(1, 99), rate=1e3, seed=2)]):
        p = tmp_path / f"t{i}.jsonl"
        save_trace(tr, p)
        a, b = load_trace(p), load_trace_json(p)
        assert (a.rate, a.seed) == (b.rate, b.seed)
        ca, cb = a.columns(), b.columns()
        for k in ("rel_id", "arrival", "output_limit", "prefix_len", "row_off", "tok", "out"):
            assert np.array_equal(getattr(ca, k), getattr(cb, k)), k
        assert ca.token_seed == cb.token_seed


@pytest.mark.parametrize("bad", [
    '{"schema": "relsim-trace-v2", "rate": 1.0, "seed": 0}\n',
    '{"schema": "relsim-trace-v1", "rate": 1.0, "seed": 0}\n{"rel_id": 0, "arrival_s": 0.5, "size": 2, '
    '"output_limit": 5, "prefix_len": 8, "requests": [{"tok": 20, "prefix_len": 8, "out": 3}]}\n',
    '{"schema": "relsim-trace-v1", "rate": 1.0, "seed": 0}\n{"rel_id": 0, "arrival_s": 0.5, "size": 1, '
    '"output_limit": 5, "prefix_len": 8, "requests": [{"tok": 20, "prefix_len": 9, "out": 3}]}\n',
    '{"schema": "relsim-trace-v1", "rate": 1.0, "seed": 0}\n{"rel_id": 0, "arrival_s": 0.5, "size": 1, ',
])
def test_native_v1_reader_rejects_malformed_files(bad, tmp_path):
    from paper_2601_11546_b200 import load_trace
    from paper_2601_11546_b200.workload import SchemaError

    p = tmp_path / "bad.jsonl"
    p.write_text(bad)
    with pytest.raises((SchemaError, ValueError)):
        load_trace(p)


def test_lazy_result_dict_behaves_like_dict():
    """RunResult.ledgers / relquery_sizes are built on first use; every dict path sees the data."""
    import json
    import pickle

    from paper_2601_11546_b200.engine import _LazyDict

    calls = []

    def build():
        calls.append(1)
        return {3: 30, 1: 10}

    d = _LazyDict(build)
    assert not calls
    assert len(d) == 2 and calls == [1]
    assert d == {3: 30, 1: 10} and dict(d) == {3: 30, 1: 10} and {**d} == {3: 30, 1: 10}
    assert sorted(d) == [1, 3] and list(d.items()) == [(3, 30), (1, 10)] and 1 in d and d.get(2) is None
    assert json.loads(json.dumps(_LazyDict(build))) == {"3": 30, "1": 10}
    assert pickle.loads(pickle.dumps(_LazyDict(build))) == {3: 30, 1: 10}
    e = _LazyDict(build)
    e[5] = 50
    assert e == {3: 30, 1: 10, 5: 50}
    assert bool(_LazyDict(dict)) is False


def test_fullscale_fingerprint_canonical():
    """The full-run fingerprints (tests/fullscale_util.py) ignore NaN payloads and
    integer widths, and the committed oracle fingerprints cover configs 2 and 3."""
    import json
    from pathlib import Path

    from fullscale_util import FIELDS, fingerprint

    from paper_2601_11546_b200 import _abi

    r1 = np.zeros(3, _abi.ITER_RECORD_DTYPE)
    r1["m_plus"] = [1.0, np.nan, 2.0]
    r2 = r1.copy()
    r2["m_plus"][1] = -np.nan  # another NaN bit pattern
    assert fingerprint(r1, np.array([1, -1], np.int32)) == fingerprint(r2, np.array([1, -1], np.int64))
    r2["m_plus"][2] = 2.0000000000000004
    assert fingerprint(r1, np.zeros(1))["sha256_m_plus"] != fingerprint(r2, np.zeros(1))["sha256_m_plus"]
    g = json.loads((Path(__file__).parent / "golden" / "fullscale.json").read_text())
    for name in ("config2", "config3"):
        assert all(f"sha256_{k}" in g["configs"][name] for k in FIELDS)
        assert g["configs"][name]["records"] == g["configs"][name]["iterations"] > 100_000


def test_run_result_to_relsim_types():
    """RunResult.to_relsim() builds the reference's own RunResult (engine.py:77-138)
    field for field; relsim itself is imported when present (build container)."""
    import math
    import sys
    from pathlib import Path

    from paper_2601_11546_b200 import engine as E

    res = E.RunResult("relserve", 1.0, 0, {7: E.TimestampLedger(0.5, 0.6, 0.7, 0.9)}, {7: 3},
                      [E.DecisionLogEntry(0, 0.0, "forced", None, None, None, None, None, "idle"),
                       E.DecisionLogEntry(1, 0.5, "transitional", 0.1, 0.2, 0.3, -0.4, -0.1, "prefill")],
                      2, 0.9, 0.0, 0.0, 5, 7)
    mods = [E]
    if Path("/root/reference/pkg/src").exists():
        sys.path.insert(0, "/root/reference/pkg/src")
        try:
            import relsim.engine as RE

            mods.append(RE)
        finally:
            sys.path.pop(0)
    for m in mods:
        r = res.to_relsim(m)
        assert type(r) is m.RunResult
        assert r.ledgers[7] == m.TimestampLedger(0.5, 0.6, 0.7, 0.9)
        assert [type(e) for e in r.decision_log] == [m.DecisionLogEntry] * 2
        assert r.decision_log[1].delta_total == -0.1 and r.decision_log[0].m_plus is None
        assert math.isclose(r.cache_hit_ratio, 5 / 12)
