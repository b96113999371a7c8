"""Generate golden fixtures by running the REAL reference engine (relsim).

Test infrastructure only.  Runs in the build container where the reference
package is mounted read-only at /root/reference (it does not exist on the GPU
box, so the fixtures are committed):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [names...]

Each fixture records, per scheduler iteration, everything the parity tests
compare bit-for-bit: the decision (case/action, m+/m-, Delta terms), the waiting
head and count, the executed prefill batch (rel_id, req_ids) or decode size,
kv_reserved after execution, the DPU's re-estimated priority values, and
(small cases) the full waiting order and the DPU RNG state; plus each
request's completion iteration and the RunResult summary/ledgers.  Traces
are described by their generator config (or an explicit spec for handmade
traces) plus a digest of their counts, so the mirror `generate_trace` is
pinned against the reference one.
"""

from __future__ import annotations

import gzip
import json
import math
import sys
import tempfile
import time
from pathlib import Path

REF_SRC = "/root/reference/pkg/src"
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, REF_SRC)
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import relsim  # noqa: E402
from relsim.cost_model import LinearCostModel, world_preset  # noqa: E402
from relsim.engine import Engine, EngineConfig, SimulationAborted  # noqa: E402
from relsim.priority import SchedulerConstraints  # noqa: E402
from relsim.workload import ArrivalTrace, RelQuery, Request, TraceConfig, generate_trace, load_trace  # noqa: E402

from golden_util import GOLDEN_DIR, SP_FNS, digest_entries  # noqa: E402

TEST_MODEL = (0.001, 0.02, 0.0002, 0.015)  # pkg/tests/test_engine.py:11


def _f(x):
    if x is None:
        return None
    if isinstance(x, float) and math.isinf(x):
        return "inf" if x > 0 else "-inf"
    return x


class Recorder(Engine):
    """Engine subclass that records per-iteration state (the CheckingEngine seam,
    pkg/tests/test_engine.py:158-176)."""

    def __init__(self, *a, full=True, **kw):
        super().__init__(*a, **kw)
        self.full = full
        self.rec = []
        self.completion = {}
        self._cur = None
        self._dpu_rows = None
        self._rng_state = None
        self.rng_initial = self.dpu.rng.bit_generator.state if self.dpu else None
        if self.dpu is not None:
            orig = self.dpu.update

            def upd(rqs, it, clock):
                recs = orig(rqs, it, clock)
                if self.full:
                    self._dpu_rows = [[rid, r.value, int(r.reused), int(r.starvation_override)]
                                      for rid, r in recs.items()]
                else:
                    self._dpu_rows = [[rid, r.value, 0, int(r.starvation_override)]
                                      for rid, r in recs.items() if not r.reused]
                st = self.dpu.rng.bit_generator.state
                self._rng_state = [str(st["state"]["state"]), int(st["has_uint32"]), int(st["uinteger"])]
                return recs

            self.dpu.update = upd

    def _flush(self):
        if self._cur is None:
            return
        cur = self._cur
        if self.config.log_decisions and len(self.decision_log) > cur["it"] - self._log_base:
            e = self.decision_log[cur["it"] - self._log_base]
            assert e.iteration == cur["it"]
            cur.update(clock=e.clock, case=e.case, action=e.action, mp=_f(e.m_plus),
                       mm=_f(e.m_minus), dp=_f(e.delta_plus), dm=_f(e.delta_minus),
                       dt=_f(e.delta_total))
        cur["kv"] = self.kv_reserved
        cur["clock_after"] = self.clock
        self.rec.append(cur)
        self._cur = None

    _log_base = 0

    def admit_arrivals(self):
        self._flush()
        n = super().admit_arrivals()
        self._cur = {"it": self.iteration, "admitted": n}
        return n

    def _update_priorities(self):
        self._dpu_rows = None
        super()._update_priorities()
        cur = self._cur
        cur["W"] = len(self.waiting)
        cur["head"] = self.waiting[0].relquery.rel_id if self.waiting else None
        if self.full:
            cur["order"] = [e.relquery.rel_id for e in self.waiting]
        if self._dpu_rows is not None:
            cur["dpu"] = self._dpu_rows
            cur["rng"] = self._rng_state

    def _execute_prefill(self, batch):
        self._cur["pb"] = [batch.requests[0].rel_id, [r.req_id for r in batch.requests]]
        return super()._execute_prefill(batch)

    def _execute_decode(self, batch):
        self._cur["nd"] = batch.num_requests
        out = super()._execute_decode(batch)
        for r in batch.requests:
            if r.done:
                key = (r.rel_id, r.req_id)
                if key not in self.completion:
                    self.completion[key] = self.iteration
        return out


def ref_trace(spec):
    kind = spec["kind"]
    if kind == "generate":
        return generate_trace(TraceConfig(**{**spec["config"], "size_range": tuple(spec["config"]["size_range"])}))
    if kind == "handmade":
        # disjoint token ranges (pkg/tests/test_engine.py:14-35)
        entries = []
        for rel_id, n, tok, limit, actual, arrival in spec["relqueries"]:
            reqs = [
                Request(rel_id=rel_id, req_id=i,
                        tokens=[1_000_000 * rel_id + 10_000 * i + j for j in range(tok)],
                        output_limit=limit,
                        actual_output_len=actual if actual is not None else limit,
                        arrival=arrival)
                for i in range(n)
            ]
            entries.append(RelQuery(rel_id=rel_id, requests=reqs, output_limit=limit, arrival=arrival))
        return ArrivalTrace(entries=entries, rate=spec.get("rate", 1.0), seed=spec.get("seed", 0))
    if kind == "heavy":
        from paper_2601_11546_b200.workload import generate_heavy_tail_trace, save_trace
        t = generate_heavy_tail_trace(**spec["config"])
        with tempfile.TemporaryDirectory() as d:
            p = Path(d) / "trace.jsonl"
            save_trace(t, p)
            return load_trace(p)
    raise ValueError(kind)


def engine_config(c):
    cc = dict(c)
    cons = cc.pop("constraints", None)
    kw = {}
    if cons:
        kw["constraints"] = SchedulerConstraints(*cons)
    if "sp_fns" in cc:
        cc["sp_priority_fns"] = SP_FNS[cc.pop("sp_fns")]
    if "tau" in cc:
        cc["tau"] = float(cc["tau"])
    kw.update(cc)
    return EngineConfig(**kw)


def model_of(m):
    if m is None:
        return None
    if isinstance(m, str):
        return world_preset(m)
    return LinearCostModel(*m)


def _csv_text(write) -> str:
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "out.csv"
        write(p)
        return p.read_text()


def run_case(name, spec, policy, world, config=None, policy_model=None, seed=0, window=None, full=True,
             csv=False):
    t0 = time.perf_counter()
    trace = ref_trace(spec)
    t_gen = time.perf_counter() - t0
    cfg = engine_config(config or {})
    if window is not None:
        cfg.iteration_limit = window
    eng = Recorder(trace, policy, model_of(world), cfg, model_of(policy_model), seed, full=full)
    aborted = None
    t0 = time.perf_counter()
    try:
        res = eng.run()
    except SimulationAborted as e:
        aborted = str(e)
        res = None
    t_run = time.perf_counter() - t0
    eng._flush()
    ledgers = {str(k): [v.arrival, v.first_prefill_start, v.last_prefill_end, v.last_decode_end]
               for k, v in eng.ledgers.items()}
    completion = {}
    for q in trace.entries:
        completion[str(q.rel_id)] = [eng.completion.get((q.rel_id, r.req_id), -1) for r in q.requests]
    if window is not None:
        # keep windowed fixtures small: only relQueries that completed something
        completion = {k: v for k, v in completion.items() if any(x >= 0 for x in v)}
    out = {
        "name": name,
        "numpy": np.__version__,
        "reference": "relsim " + getattr(relsim, "__version__", "?"),
        "trace": spec,
        "trace_digest": digest_entries(trace.entries),
        "num_requests": trace.num_requests,
        "policy": policy,
        "world": world,
        "policy_model": policy_model,
        "config": config or {},
        "seed": seed,
        "window": window,
        "aborted": aborted,
        "rng_initial": None if eng.rng_initial is None else {
            "state": str(eng.rng_initial["state"]["state"]),
            "inc": str(eng.rng_initial["state"]["inc"]),
            "has_uint32": int(eng.rng_initial["has_uint32"]),
            "uinteger": int(eng.rng_initial["uinteger"]),
        },
        "result": {
            "iterations": eng.iteration,
            "sim_duration": eng.clock,
            "cache_hit_tokens": eng.cache.hit_tokens_total,
            "cache_miss_tokens": eng.cache.miss_tokens_total,
            "kv_reserved": eng.kv_reserved,
            "decision_log_len": len(eng.decision_log),
        },
        "ledgers": ledgers,
        "completion": completion,
        "iters": eng.rec,
        "timing": {"trace_s": t_gen, "run_s": t_run},
    }
    if csv and res is not None:  # RunResult CSVs (engine.py:104-138), byte for byte
        out["csv"] = {"relquery": _csv_text(res.write_relquery_csv), "decision": _csv_text(res.write_decision_csv)}
    p = GOLDEN_DIR / f"{name}.json.gz"
    with gzip.open(p, "wt", compresslevel=9) as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"{name}: iters={eng.iteration} run={t_run:.2f}s gen={t_gen:.1f}s -> {p.stat().st_size} B", flush=True)


def gen(cfg):
    return {"kind": "generate", "config": cfg}


CFG1 = gen({"num_relqueries": 8, "size_range": [100, 100], "rate": 1.0, "seed": 0})
STARVE = {"kind": "handmade", "relqueries": [[0, 40, 150, 50, None, 0.0]]
          + [[i, 1, 50, 5, None, 0.1 * (i - 1)] for i in range(1, 61)]}
HOL = {"kind": "handmade", "relqueries": [[0, 60, 150, 50, None, 0.0], [1, 2, 50, 3, None, 0.0]]}
TIGHT = {"constraints": [4000, 16, 512]}

CASES = {
    # config 1: all five policies
    "cfg1_relserve": dict(spec=CFG1, csv=True, policy="relserve", world="opt-13b-like"),
    "cfg1_fcfs": dict(spec=CFG1, csv=True, policy="fcfs", world="opt-13b-like"),
    "cfg1_sp": dict(spec=CFG1, csv=True, policy="sp", world="opt-13b-like"),
    "cfg1_pp": dict(spec=CFG1, csv=True, policy="relserve-pp", world="opt-13b-like"),
    "cfg1_dp": dict(spec=CFG1, csv=True, policy="relserve-dp", world="opt-13b-like"),
    # sp with user priority functions of either sign (priority.py:221-235)
    "sp_negative": dict(spec=gen({"num_relqueries": 30, "size_range": [1, 40], "rate": 4.0, "seed": 41}),
                        policy="sp", world="opt-13b-like", config={"sp_fns": "neg_mixed"}),
    "sp_negative_only": dict(spec=gen({"num_relqueries": 25, "size_range": [1, 30], "rate": 6.0, "seed": 42}),
                             policy="sp", world=list(TEST_MODEL), config={"sp_fns": "neg_only"}),
    # tight constraints (pkg/tests/test_engine.py:181-195)
    "tight_relserve": dict(spec=gen({"num_relqueries": 25, "size_range": [1, 30], "rate": 5.0, "seed": 21}),
                           policy="relserve", world=list(TEST_MODEL), config=TIGHT),
    "tight_fcfs": dict(spec=gen({"num_relqueries": 25, "size_range": [1, 30], "rate": 5.0, "seed": 21}),
                       policy="fcfs", world=list(TEST_MODEL), config=TIGHT),
    # prefix-cache eviction pressure
    "evict_relserve": dict(spec=gen({"num_relqueries": 40, "size_range": [1, 40], "rate": 3.0, "seed": 5}),
                           policy="relserve", world="opt-13b-like", config={"capacity_blocks": 64}),
    "evict_tiny": dict(spec=gen({"num_relqueries": 30, "size_range": [1, 25], "rate": 8.0, "seed": 17}),
                       policy="relserve", world="qwen-32b-like",
                       config={"capacity_blocks": 24, "constraints": [20000, 48, 2048]}),
    "evict_block8": dict(spec=gen({"num_relqueries": 30, "size_range": [1, 25], "rate": 2.0, "seed": 23,
                                   "mean_input_len": 90}),
                         policy="relserve-pp", world="opt-13b-like",
                         config={"capacity_blocks": 100, "block_size": 8, "sample_size": 3}),
    # truncated inserts: rows with more whole blocks than the whole cache (prefix_cache.py:101-103)
    "evict_truncate": dict(spec=gen({"num_relqueries": 20, "size_range": [1, 20], "rate": 3.0, "seed": 29}),
                           policy="relserve", world="opt-13b-like", config={"capacity_blocks": 10}),
    "evict_truncate_fcfs": dict(spec=gen({"num_relqueries": 15, "size_range": [1, 12], "rate": 5.0, "seed": 30,
                                          "mean_input_len": 300}),
                                policy="fcfs", world="opt-13b-like", config={"capacity_blocks": 14}),
    # starvation override
    "tau_relserve": dict(spec=gen({"num_relqueries": 40, "size_range": [1, 60], "rate": 2.0, "seed": 11}),
                         policy="relserve", world=list(TEST_MODEL), config={"tau": 0.05}, csv=True),
    "starve_tau": dict(spec=STARVE, policy="relserve", world=list(TEST_MODEL), config={"tau": 0.05}),
    "starve_inf": dict(spec=STARVE, policy="relserve", world=list(TEST_MODEL)),
    "hol_relserve": dict(spec=HOL, policy="relserve", world=list(TEST_MODEL)),
    "hol_fcfs": dict(spec=HOL, policy="fcfs", world=list(TEST_MODEL)),
    # belief != world, other sample size / seed
    "mismatch_relserve": dict(spec=gen({"num_relqueries": 30, "size_range": [1, 50], "rate": 1.5, "seed": 3}),
                              policy="relserve", world="opt-13b-like", policy_model="qwen-32b-like",
                              config={"sample_size": 4}, seed=3),
    # paper-scale trace (100 relQ x U[1,100])
    "paper_relserve": dict(spec=gen({"num_relqueries": 100, "size_range": [1, 100], "rate": 1.0, "seed": 0}),
                           policy="relserve", world="opt-13b-like", full=False),
    "paper_dp": dict(spec=gen({"num_relqueries": 100, "size_range": [1, 100], "rate": 0.5, "seed": 1}),
                     policy="relserve-dp", world="opt-13b-like", full=False),
    # config-4 cells (100 relQ, sizes (1,s), seed = cell index)
    "cfg4_cell_a": dict(spec=gen({"num_relqueries": 100, "size_range": [1, 8], "rate": 4.0, "seed": 7}),
                        policy="relserve", world="llama-70b-like", full=False),
    "cfg4_cell_b": dict(spec=gen({"num_relqueries": 100, "size_range": [1, 64], "rate": 0.25, "seed": 300}),
                        policy="relserve", world="opt-13b-like", full=False),
    # world-model noise (engine.py:310-313): noisy batch durations
    "noise_relserve": dict(spec=gen({"num_relqueries": 40, "size_range": [1, 60], "rate": 2.0, "seed": 13}),
                           policy="relserve", world="opt-13b-like", config={"noise_sigma": 0.1}, seed=4),
    "noise_fcfs": dict(spec=gen({"num_relqueries": 30, "size_range": [1, 40], "rate": 3.0, "seed": 14}),
                       policy="fcfs", world=list(TEST_MODEL), config={"noise_sigma": 0.5}, seed=2),
    # configs 2 / 3: windowed (first 40 iterations)
    "cfg2_window": dict(spec=gen({"num_relqueries": 1000, "size_range": [1000, 1000], "rate": 1e6, "seed": 0}),
                        policy="relserve", world="opt-13b-like", window=40),
    "cfg3_window": dict(spec={"kind": "heavy", "config": {"num_relqueries": 5000, "size_range": [1, 399],
                                                           "rate": 1e6, "seed": 0}},
                        policy="relserve", world="llama-70b-like", window=40),
}


#: report.summarize (report.py:101-155) over full reference runs: (trace spec, policy, world) each;
#: config 1 at two rates under every policy, so speedups vs fcfs exist at both rates
SUMMARY_RUNS = [(gen({"num_relqueries": 8, "size_range": [100, 100], "rate": r, "seed": 0}), p, "opt-13b-like")
                for r in (1.0, 2.0) for p in ("fcfs", "sp", "relserve", "relserve-pp", "relserve-dp")]


def make_summary():
    """tests/golden/summary.json: the summary tables' CSV bytes (wide and long, baselines fcfs
    and sp) and each run's ledgers and sizes, for the report parity tests."""
    from relsim.report import summarize

    runs, rows = [], []
    for spec, policy, world in SUMMARY_RUNS:
        res = Engine(ref_trace(spec), policy, model_of(world), EngineConfig(), None, 0).run()
        runs.append(res)
        rows.append({"spec": spec, "policy": policy, "world": world, "rate": res.rate,
                     "ledgers": [[k, v.arrival, v.first_prefill_start, v.last_prefill_end, v.last_decode_end]
                                 for k, v in res.ledgers.items()],
                     "sizes": [[k, v] for k, v in res.relquery_sizes.items()]})
    out = {"numpy": np.__version__, "reference": "relsim " + getattr(relsim, "__version__", "?"), "runs": rows,
           "tables": {}}
    for base in ("fcfs", "sp"):
        t = summarize(runs, baseline=base)
        out["tables"][base] = {"wide": _csv_text(t.write_csv), "long": _csv_text(t.write_long_csv)}
    p = GOLDEN_DIR / "summary.json"
    p.write_text(json.dumps(out, indent=1) + "\n")
    print(f"summary: {len(runs)} runs -> {p.stat().st_size} B")


def main(argv):
    GOLDEN_DIR.mkdir(parents=True, exist_ok=True)
    if argv == ["summary"]:
        make_summary()
        return
    names = argv or [n for n in CASES if not n.startswith(("cfg2", "cfg3"))]
    for n in names:
        run_case(n, **CASES[n])


if __name__ == "__main__":
    main(sys.argv[1:])
