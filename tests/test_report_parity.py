"""RunResult CSVs and report.summarize byte for byte against the reference
(SURVEY 8(f)3): the reference's own writers' output is recorded in the goldens
(tests/golden/make_golden.py: `csv` of the cfg1_* / tau_relserve fixtures and
tests/golden/summary.json).  CPU tests rebuild RunResults from the recorded
ledgers and decisions; the GPU tests write the device runs' own results."""

import json
import math
import tempfile
from pathlib import Path

import pytest

import parity
from golden_util import GOLDEN_DIR, golden_names, load_golden

CSV_GOLDENS = [n for n in golden_names() if "csv" in load_golden(n)]
SUMMARY = json.loads((GOLDEN_DIR / "summary.json").read_text())


def _text(write) -> str:
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "out.csv"
        write(p)
        return p.read_text()


def _fl(x):
    return None if x is None else float(x)


def _result_from_golden(g):
    """A mirror RunResult carrying the reference run's ledgers (in the reference's dict order),
    sizes and decision log."""
    from paper_2601_11546_b200.engine import DecisionLogEntry, RunResult, TimestampLedger

    trace = parity.build_trace(g["trace"])
    c = trace.columns()
    sizes = dict(zip(c.rel_id.tolist(), [int(x) for x in (c.row_off[1:] - c.row_off[:-1])]))
    ledgers = {int(k): TimestampLedger(*(_fl(x) for x in v)) for k, v in g["ledgers"].items()}
    log = [DecisionLogEntry(e["it"], e["clock"], e["case"], _fl(e["mp"]), _fl(e["mm"]), _fl(e["dp"]), _fl(e["dm"]),
                            _fl(e["dt"]), e["action"]) for e in g["iters"]]
    r = g["result"]
    return RunResult(g["policy"], trace.rate, g["seed"], ledgers, {k: sizes[k] for k in ledgers}, log,
                     r["iterations"], r["sim_duration"], 0.0, 0.0, r["cache_hit_tokens"], r["cache_miss_tokens"])


def _summary_runs():
    from paper_2601_11546_b200.engine import RunResult, TimestampLedger

    out = []
    for run in SUMMARY["runs"]:
        ledgers = {int(k): TimestampLedger(a, b, c, d) for k, a, b, c, d in run["ledgers"]}
        out.append(RunResult(run["policy"], run["rate"], 0, ledgers, {int(k): v for k, v in run["sizes"]}, [],
                             0, 0.0, 0.0, 0.0, 0, 0))
    return out


def test_goldens_carry_csvs():
    assert {"cfg1_relserve", "cfg1_fcfs", "cfg1_sp", "cfg1_pp", "cfg1_dp", "tau_relserve"} <= set(CSV_GOLDENS)


@pytest.mark.parametrize("name", CSV_GOLDENS)
def test_run_result_csvs_match_reference_bytes(name):
    g = load_golden(name)
    res = _result_from_golden(g)
    assert _text(res.write_relquery_csv) == g["csv"]["relquery"]
    assert _text(res.write_decision_csv) == g["csv"]["decision"]


@pytest.mark.parametrize("baseline", ["fcfs", "sp"])
def test_summarize_matches_reference_bytes(baseline):
    from paper_2601_11546_b200.report import summarize

    t = summarize(_summary_runs(), baseline=baseline)
    want = SUMMARY["tables"][baseline]
    assert _text(t.write_csv) == want["wide"]
    assert _text(t.write_long_csv) == want["long"]


def test_summarize_errors_and_nan_speedup():
    from paper_2601_11546_b200.report import summarize

    runs = _summary_runs()
    with pytest.raises(ValueError):
        summarize([])
    t = summarize([r for r in runs if r.policy != "fcfs"], baseline="fcfs")
    assert all(math.isnan(row.speedup_vs_baseline) for row in t.rows)
    other = _summary_runs()[0]
    other.ledgers.pop(next(iter(other.ledgers)))
    with pytest.raises(ValueError):
        summarize([runs[1], other])


@pytest.mark.gpu
@pytest.mark.parametrize("name", CSV_GOLDENS)
def test_device_run_csvs_match_reference_bytes(name):
    from paper_2601_11546_b200.engine import Engine

    g = load_golden(name)
    trace, policy, world, cfg, pm, seed = parity.golden_inputs(g)
    eng = Engine(trace, policy, world, cfg, pm, seed, device=0)
    res = eng.run()
    eng.close()
    assert _text(res.write_relquery_csv) == g["csv"]["relquery"]
    assert _text(res.write_decision_csv) == g["csv"]["decision"]


@pytest.mark.gpu
def test_device_runs_summarize_to_reference_bytes():
    """Average relQuery latency parity end to end: the reference's summary tables from the
    device's own runs of the same traces."""
    from paper_2601_11546_b200 import summarize
    from paper_2601_11546_b200.engine import Engine, EngineConfig

    runs = []
    for run in SUMMARY["runs"]:
        trace = parity.build_trace(run["spec"])
        eng = Engine(trace, run["policy"], parity.model_of(run["world"]), EngineConfig(), None, 0, device=0)
        runs.append(eng.run())
        eng.close()
    for base, want in SUMMARY["tables"].items():
        t = summarize(runs, baseline=base)
        assert _text(t.write_csv) == want["wide"]
        assert _text(t.write_long_csv) == want["long"]
