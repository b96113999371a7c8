"""Parity helpers: rebuild golden inputs with the mirror types and compare runs.

Test infrastructure only.
"""

from __future__ import annotations

import math

import numpy as np

from golden_util import SP_FNS, digest_columns
from paper_2601_11546_b200 import _abi
from paper_2601_11546_b200.cost_model import LinearCostModel, world_preset
from paper_2601_11546_b200.engine import EngineConfig
from paper_2601_11546_b200.priority import SchedulerConstraints
from paper_2601_11546_b200.workload import (
    ArrivalTrace, RelQuery, Request, TraceConfig, generate_heavy_tail_trace, generate_trace)


def build_trace(spec) -> ArrivalTrace:
    kind = spec["kind"]
    if kind == "generate":
        cfg = dict(spec["config"])
        cfg["size_range"] = tuple(cfg["size_range"])
        return generate_trace(TraceConfig(**cfg))
    if kind == "handmade":
        entries = []
        for rel_id, n, tok, limit, actual, arrival in spec["relqueries"]:
            reqs = [Request(rel_id, i, [1_000_000 * rel_id + 10_000 * i + j for j in range(tok)],
                            limit, actual if actual is not None else limit, arrival)
                    for i in range(n)]
            entries.append(RelQuery(rel_id, reqs, limit, arrival))
        return ArrivalTrace(entries, spec.get("rate", 1.0), spec.get("seed", 0))
    if kind == "heavy":
        return generate_heavy_tail_trace(**spec["config"])
    raise ValueError(kind)


def model_of(m):
    if m is None:
        return None
    if isinstance(m, str):
        return world_preset(m)
    return LinearCostModel(*m)


def engine_config(c: dict, window=None) -> EngineConfig:
    c = dict(c)
    kw = {}
    cons = c.pop("constraints", None)
    if cons:
        kw["constraints"] = SchedulerConstraints(*cons)
    if "sp_fns" in c:
        c["sp_priority_fns"] = SP_FNS[c.pop("sp_fns")]
    if "tau" in c:
        c["tau"] = float(c["tau"])
    kw.update(c)
    cfg = EngineConfig(**kw)
    if window is not None:
        cfg.iteration_limit = window
    return cfg


def golden_inputs(g):
    trace = build_trace(g["trace"])
    assert digest_columns(trace.columns()) == g["trace_digest"], "mirror trace != reference trace"
    return (trace, g["policy"], model_of(g["world"]), engine_config(g["config"], g["window"]),
            model_of(g["policy_model"]), g["seed"])


def _fl(x):
    if x is None:
        return math.nan
    if x == "inf":
        return math.inf
    return float(x)


def _same(a: float, b: float) -> bool:
    return (math.isnan(a) and math.isnan(b)) or a == b


def compare_records(recs: np.ndarray, g, trace: ArrivalTrace, what: str = "run"):
    """Bit-exact comparison of rs_iter_record rows against a golden's iterations."""
    c = trace.columns()
    rel = c.rel_id
    gi = g["iters"]
    assert len(recs) == len(gi), f"{what}: {len(recs)} iterations vs golden {len(gi)}"
    for r, e in zip(recs, gi):
        it = int(r["iteration"])
        ctx = f"{what} iteration {it}"
        assert it == e["it"], ctx
        assert r["clock"] == e["clock"], f"{ctx}: clock {r['clock']!r} != {e['clock']!r}"
        assert _abi.ACTIONS[r["action"]] == e["action"], f"{ctx}: action"
        assert _abi.CASES[r["kase"]] == e["case"], f"{ctx}: case {_abi.CASES[r['kase']]} != {e['case']}"
        for k, gk in (("m_plus", "mp"), ("m_minus", "mm"), ("delta_plus", "dp"),
                      ("delta_minus", "dm"), ("delta_total", "dt")):
            assert _same(float(r[k]), _fl(e[gk])), f"{ctx}: {k} {r[k]!r} != {e[gk]!r}"
        head = None if r["head"] < 0 else int(rel[r["head"]])
        assert head == e["head"], f"{ctx}: head {head} != {e['head']}"
        assert int(r["n_waiting"]) == e["W"], f"{ctx}: W {r['n_waiting']} != {e['W']}"
        if "pb" in e:
            assert r["batch_rq"] >= 0 and int(rel[r["batch_rq"]]) == e["pb"][0], f"{ctx}: batch rq"
            ids = list(range(int(r["batch_first"]), int(r["batch_first"]) + int(r["batch_n"])))
            assert ids == e["pb"][1], f"{ctx}: batch {ids} != {e['pb'][1]}"
        elif "nd" in e:
            assert int(r["batch_n"]) == e["nd"], f"{ctx}: decode n {r['batch_n']} != {e['nd']}"
        assert int(r["kv_reserved"]) == e["kv"], f"{ctx}: kv {r['kv_reserved']} != {e['kv']}"


def compare_completion(comp: np.ndarray, g, trace: ArrivalTrace):
    c = trace.columns()
    off = c.row_off
    idx = {int(r): i for i, r in enumerate(c.rel_id.tolist())}
    for rid, lst in g["completion"].items():
        i = idx[int(rid)]
        got = comp[off[i]:off[i + 1]].tolist()
        assert got == lst, f"completion iterations of relQuery {rid} differ"
    if g["window"] is None:
        # every request completes in a full run
        assert int((comp < 0).sum()) == 0


def compare_ledgers(fps, lpe, lde, g, trace: ArrivalTrace):
    c = trace.columns()
    idx = {int(r): i for i, r in enumerate(c.rel_id.tolist())}
    for rid, (arr, a, b, d) in g["ledgers"].items():
        i = idx[int(rid)]
        for got, want, name in ((fps[i], a, "first_prefill_start"), (lpe[i], b, "last_prefill_end"),
                                (lde[i], d, "last_decode_end")):
            assert _same(float(got), _fl(want)), f"ledger {rid}.{name}: {got!r} != {want!r}"


def golden_dpu_by_iter(g):
    """{iteration: {rel_id: value}} of re-estimated (non-reused) DPU records."""
    out = {}
    for e in g["iters"]:
        if "dpu" in e:
            out[e["it"]] = {rid: val for rid, val, reused, ov in e["dpu"] if not reused}
    return out


def compare_priority_records(res, g, what: str = "run") -> int:
    """Device DPU records (RunResult.priority_records, parity mode) against the golden's
    `dpu` rows (priority.py:287-315: value, reused, starvation_override per live relQuery in
    dict order; only the recomputed ones in fixtures recorded with full=False) and the DPU
    generator state after each update.  Values compare bit for bit.  Returns the iterations
    checked."""
    n = 0
    for i, e in enumerate(g["iters"]):
        if "dpu" not in e:
            continue
        pr = res.priority_records[i]
        full = any(row[2] for row in e["dpu"]) or len(e["dpu"]) == len(pr.rel_id)
        rows = [[int(r), float(v), int(u), int(o)] for r, v, u, o in
                zip(pr.rel_id.tolist(), pr.value.tolist(), pr.reused.tolist(), pr.starvation_override.tolist())]
        if not full:
            rows = [[r, v, 0, o] for r, v, u, o in rows if not u]
        want = [[int(r), float(v), int(u), int(o)] for r, v, u, o in e["dpu"]]
        assert rows == want, f"{what}: DPU records differ at iteration {e['it']}: " + next(
            (f"{a} != {b}" for a, b in zip(rows, want) if a != b), f"{len(rows)} vs {len(want)} records")
        st, has, u = res.dpu_rng_states[i]
        assert [str(st), has, u] == e["rng"], f"{what}: DPU RNG state differs at iteration {e['it']}"
        n += 1
    return n
