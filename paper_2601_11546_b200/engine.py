"""GPU-resident scheduling engine: drop-in for `relsim.engine` (engine.py:45-475).

`run(trace, policy, world_model, config, policy_model, seed) -> RunResult` and
`Engine(...)` keep the reference signatures.  Every scheduler iteration --
admission, the Dynamic Priority Updater with its PEM estimator and numpy
PCG64 sample replay, the waiting-queue order, the Adaptive Batch Arranger
with the Delta projection, and the prefill/decode/idle state advance with the
prefix-cache model -- runs on the GPU inside one persistent sm_100a kernel
per trace (paper_2601_11546_b200/csrc/engine.cu).  The host only uploads the
trace columns, launches chunks of iterations and copies back the decision
records, ledgers and per-request state.  There is no CPU fallback: if the
CUDA library is missing or the GPU is absent, construction fails.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _abi, _marshal
from .cost_model import LinearCostModel
from .priority import InfeasibleRequestError, SchedulerConstraints
from .workload import ArrivalTrace

POLICIES = ("fcfs", "sp", "relserve", "relserve-pp", "relserve-dp")


class SimulationAborted(RuntimeError):
    pass


@dataclass
class TimestampLedger:
    arrival: float
    first_prefill_start: float | None = None
    last_prefill_end: float | None = None
    last_decode_end: float | None = None

    @property
    def complete(self) -> bool:
        return self.last_decode_end is not None


@dataclass
class DecisionLogEntry:
    iteration: int
    clock: float
    case: str
    m_plus: float | None
    m_minus: float | None
    delta_plus: float | None
    delta_minus: float | None
    delta_total: float | None
    action: str


@dataclass
class RunResult:
    """Mirror of relsim's RunResult (engine.py:77-138) plus device-side extras."""

    policy: str
    rate: float
    seed: int
    ledgers: dict[int, TimestampLedger]
    relquery_sizes: dict[int, int]
    decision_log: list[DecisionLogEntry]
    iterations: int
    sim_duration: float
    dpu_wall_s: float
    aba_wall_s: float
    cache_hit_tokens: int
    cache_miss_tokens: int
    #: per request (trace order): iteration of the decode that completed it, -1 if none
    completion_iteration: np.ndarray | None = None
    #: raw per-iteration records (include/relserve.h rs_iter_record)
    records: np.ndarray | None = None
    #: wall time of the whole device run (host view, includes launches/copies)
    device_wall_s: float = 0.0
    #: parity mode (Engine(record_waiting_order=True)): per iteration, the waiting queue after the
    #: priority update as trace-order relQuery indices (engine.py:277-281)
    waiting_orders: list | None = None
    #: parity mode, DPU policies: per iteration, DynamicPriorityUpdater.update's records
    #: (priority.py:287-315) in live-relQuery order -- PriorityRecords(rel_id, value, reused,
    #: starvation_override), numpy columns -- and the DPU generator state after the update
    #: ((state, has_uint32, uinteger), numpy's bit_generator.state fields)
    priority_records: list | None = None
    dpu_rng_states: list | None = None

    @property
    def cache_hit_ratio(self) -> float:
        total = self.cache_hit_tokens + self.cache_miss_tokens
        return self.cache_hit_tokens / total if total else 0.0

    @property
    def scheduler_overhead_fraction(self) -> float:
        if self.sim_duration <= 0:
            return 0.0
        return (self.dpu_wall_s + self.aba_wall_s) / self.sim_duration

    def to_relsim(self, engine_module=None):
        """The same result as a genuine ``relsim.engine.RunResult`` (engine.py:77-138), for
        callers that type-check or pickle relsim objects.  ``engine_module`` defaults to
        ``relsim.engine`` (imported on demand; this package never needs relsim itself)."""
        if engine_module is None:
            import importlib

            engine_module = importlib.import_module("relsim.engine")
        L, D = engine_module.TimestampLedger, engine_module.DecisionLogEntry
        return engine_module.RunResult(
            policy=self.policy, rate=self.rate, seed=self.seed,
            ledgers={k: L(v.arrival, v.first_prefill_start, v.last_prefill_end, v.last_decode_end)
                     for k, v in self.ledgers.items()},
            relquery_sizes=dict(self.relquery_sizes),
            decision_log=[D(e.iteration, e.clock, e.case, e.m_plus, e.m_minus, e.delta_plus, e.delta_minus,
                            e.delta_total, e.action) for e in self.decision_log],
            iterations=self.iterations, sim_duration=self.sim_duration, dpu_wall_s=self.dpu_wall_s,
            aba_wall_s=self.aba_wall_s, cache_hit_tokens=self.cache_hit_tokens,
            cache_miss_tokens=self.cache_miss_tokens)

    def write_relquery_csv(self, path) -> None:
        """Per-relQuery latency breakdown in rel_id order, floats as repr (engine.py:104-125)."""
        import csv
        from pathlib import Path

        from .report import decompose

        def rows():
            for rel_id in sorted(self.ledgers):
                led = self.ledgers[rel_id]
                b = decompose(rel_id, led)
                yield [rel_id, self.relquery_sizes[rel_id],
                       *map(repr, (led.arrival, b.waiting_s, b.core_s, b.tail_s, b.total_s))]

        with Path(path).open("w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["rel_id", "size", "arrival_s", "waiting_s", "core_s", "tail_s", "total_s"])
            w.writerows(rows())

    def write_decision_csv(self, path) -> None:
        """One row per logged iteration; None fields empty (engine.py:127-138)."""
        import csv
        from pathlib import Path

        with Path(path).open("w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["iteration", "clock_s", "case", "m_plus", "m_minus", "delta_plus", "delta_minus",
                        "delta_total", "action"])
            w.writerows([e.iteration, repr(e.clock), e.case, e.m_plus, e.m_minus, e.delta_plus, e.delta_minus,
                         e.delta_total, e.action] for e in self.decision_log)


@dataclass
class PriorityRecords:
    """One iteration's DPU records as columns (priority.py:62-68), live relQueries in
    admission order (the reference's dict order)."""

    rel_id: np.ndarray
    value: np.ndarray
    reused: np.ndarray
    starvation_override: np.ndarray


@dataclass
class EngineConfig:
    """Mirror of relsim's EngineConfig (engine.py:141-158)."""

    constraints: SchedulerConstraints = field(
        default_factory=lambda: SchedulerConstraints(
            cap=200_000, max_num_seqs=256, max_num_batched_tokens=8192
        )
    )
    noise_sigma: float = 0.0
    sample_size: int = 8
    tau: float = math.inf
    block_size: int = 16
    capacity_blocks: int = 8192
    iteration_limit: int = 5_000_000
    log_decisions: bool = True
    sp_priority_fns: tuple | None = None


def _opt(x: float):
    return None if math.isnan(x) else float(x)


#: rs_trace_status.phase_cycles slots of the priority update (DPU) and of the
#: waiting order + candidates + decision (ABA), mirroring the reference's
#: dpu_wall / aba_wall timers (engine.py:381-417); see csrc phase_mark calls
_DPU_PHASES = (1, 5, 6, 7, 8, 15, 16, 17, 18)
_ABA_PHASES = (2, 3, 11, 12)


class _DecisionLog(list):
    """RunResult.decision_log (engine.py:64-74, 419-433): a list of
    DecisionLogEntry built from the device records -- at once for logs up to
    `EAGER` entries, else on first use (every list method, comparison and
    mutator fills it first)."""

    EAGER = 1024

    def __init__(self, recs: np.ndarray):
        super().__init__()
        self._recs = recs
        if recs is None or len(recs) <= self.EAGER:
            self._fill()

    def _fill(self):
        recs, self._recs = self._recs, None
        if recs is None or not len(recs):
            return
        cols = [recs[k].tolist() for k in ("iteration", "clock", "kase", "m_plus", "m_minus", "delta_plus",
                                           "delta_minus", "delta_total", "action")]
        nan = math.isnan
        out = []
        for it, clk, ks, mp, mm, dp, dm, dt, ac in zip(*cols):
            proj = not nan(dp)
            out.append(DecisionLogEntry(
                it, clk, _abi.CASES[ks], None if nan(mp) else mp, None if nan(mm) else mm,
                dp if proj else None, dm if proj else None, dt if proj else None, _abi.ACTIONS[ac]))
        list.extend(self, out)

    def _ready(self):
        if self._recs is not None:
            self._fill()


for _name in ("__len__", "__iter__", "__getitem__", "__contains__", "__eq__", "__ne__", "__lt__", "__le__",
              "__gt__", "__ge__", "__repr__", "__reversed__", "__bool__", "index", "count", "copy", "__add__",
              "__radd__", "__mul__", "__rmul__", "__iadd__", "__imul__", "__setitem__", "__delitem__", "append",
              "extend", "clear", "sort", "insert", "pop", "remove", "reverse", "__reduce_ex__", "__sizeof__"):
    if hasattr(list, _name):
        def _wrap(name=_name):
            base = getattr(list, name)

            def f(self, *a, **k):
                self._ready()
                return base(self, *a, **k)

            f.__name__ = name
            return f

        setattr(_DecisionLog, _name, _wrap())


class _LazyDict(dict):
    """RunResult.ledgers / relquery_sizes: a dict built from the arrays already read
    back from the device on first use (10^4-10^5 Python objects are host work the
    caller may never need)."""

    _PENDING = object()  # C-level readers that test the size first (json) see a non-empty dict

    def __init__(self, build):
        super().__init__({_LazyDict._PENDING: None})
        self._build = build

    def _ready(self):
        if self._build is not None:
            build, self._build = self._build, None
            dict.clear(self)
            dict.update(self, build())


for _name in ("__len__", "__iter__", "__getitem__", "__contains__", "__eq__", "__ne__", "__repr__", "__reversed__",
              "__or__", "__ror__", "__ior__", "__setitem__", "__delitem__", "keys", "values", "items", "get", "copy",
              "pop", "popitem", "setdefault", "update", "clear"):
    if hasattr(dict, _name):
        def _wrap_d(name=_name):
            base = getattr(dict, name)

            def f(self, *a, **k):
                self._ready()
                return base(self, *a, **k)

            f.__name__ = name
            return f

        setattr(_LazyDict, _name, _wrap_d())
_LazyDict.__reduce__ = lambda self: (self._ready(), (dict, (dict.copy(self),)))[1]


_ERRORS = {
    _abi.RS_EINVAL: ValueError,
    _abi.RS_EINFEASIBLE: InfeasibleRequestError,
    _abi.RS_EABORT_LIMIT: SimulationAborted,
    _abi.RS_EABORT_IDLE: SimulationAborted,
    _abi.RS_ECACHE_PINNED: RuntimeError,
    _abi.RS_EUNSUPPORTED: NotImplementedError,
}


def raise_for(code: int, msg: str):
    if code in (_abi.RS_OK, _abi.RS_RUNNING):
        return
    raise _ERRORS.get(code, RuntimeError)(msg)


class WaitingEntry:
    """relsim's _WaitingEntry (engine.py:160-176): a relQuery's not-yet-prefilled requests."""

    __slots__ = ("relquery", "pending", "arrival_index", "_priority")

    def __init__(self, relquery, arrival_index: int):
        self.relquery = relquery
        self.pending = list(relquery.requests)
        self.arrival_index = arrival_index
        self._priority = 0.0

    @property
    def priority(self) -> float:
        return self._priority if self.pending else 0.0

    def sort_key(self):
        return (self.priority, self.relquery.arrival, self.relquery.rel_id)


class Engine:
    """Reference-signature engine whose loop runs on the GPU (engine.py:179-463)."""

    #: iterations launched per device step (one persistent-kernel launch)
    chunk_iterations = 1 << 14
    #: world-model noise draws handed to the device first (the prefix doubles when used up)
    noise_chunk = 1 << 14

    def __init__(
        self,
        trace: ArrivalTrace,
        policy: str,
        world_model: LinearCostModel,
        config: EngineConfig | None = None,
        policy_model: LinearCostModel | None = None,
        seed: int = 0,
        *,
        device: int = 0,
        stream=None,
        shards: int = 1,
        shard_rank: int = -1,
        record_waiting_order: bool = False,
    ):
        """shards > 1 runs the sharded pool (include/relserve.h rs_engine_create_sharded):
        shard_rank -1 puts every shard on `device` (one CTA each); shard_rank >= 0 makes this
        engine one shard of a multi-process group (call connect_shards before run/step).
        record_waiting_order (parity mode): also record, for every iteration, the priority
        update (RunResult.priority_records, dpu_rng_states) and the full sorted waiting queue
        (RunResult.waiting_orders, rebuilt from the priorities by the device radix sort); the
        timed path never sorts."""
        if policy not in POLICIES:
            raise ValueError(f"unknown policy {policy!r}; choose from {POLICIES}")
        self.trace = trace
        self.policy = policy
        self.world_model = world_model
        self.policy_model = policy_model if policy_model is not None else world_model
        self.config = config or EngineConfig()
        self.seed = seed
        self.device = device
        self.stream = stream
        c = self.config
        if policy in ("relserve", "relserve-pp", "relserve-dp") and not (c.tau > 0):
            raise ValueError("tau must be positive")
        if c.noise_sigma < 0:
            raise ValueError("noise_sigma must be non-negative")
        from . import _native

        self._m = _marshal.marshal_trace(trace, c.block_size, policy, self.policy_model,
                                         c.sp_priority_fns)
        self._record_order = bool(record_waiting_order and c.log_decisions)
        if self._record_order:  # parity snapshots: log capacity x relQueries cells, read after each launch
            R = max(1, trace.columns().num_relqueries)
            self.chunk_iterations = max(16, min(Engine.chunk_iterations, 1 << max(4, ((1 << 24) // R).bit_length() - 1)))
        self._native = _native.NativeEngine(
            [self._m.view], _marshal.make_config(c, policy, record_waiting_order and c.log_decisions),
            _marshal.make_model(world_model),
            _marshal.make_model(self.policy_model), [_marshal.dpu_rng_state(seed)], device,
            log_capacity=self.chunk_iterations if c.log_decisions else 0, shards=shards, rank=shard_rank,
        )
        self.shards, self.shard_rank = shards, shard_rank
        self._orders: list[np.ndarray] = []
        self._dpu_snaps: list = []
        # world-model noise (engine.py:198, 310-313): the reference's standard normals, one per
        # executed batch, from the same stream; handed to the device in growing prefixes
        self._noise_rng = None
        self._noise = np.zeros(0)
        if c.noise_sigma > 0:
            self._noise_rng = np.random.default_rng(np.random.SeedSequence([seed, 0xE7]))
            self._extend_noise(self.noise_chunk)
        self.iteration = 0
        self.clock = 0.0
        self.kv_reserved = 0
        self._records: list[np.ndarray] = []
        self._status = None
        self.result: RunResult | None = None

    # -- sharded pool across processes ----------------------------------------

    def mailbox_handle(self) -> bytes:
        """CUDA IPC handle of this shard's mailbox (shard_rank >= 0)."""
        return self._native.mailbox_handle()

    def connect_shards(self, handles: list[bytes]) -> None:
        """handles[r] = shard r's mailbox_handle(), gathered from every process."""
        self._native.connect(handles)

    # -- device loop ---------------------------------------------------------

    def _extend_noise(self, n: int) -> None:
        self._noise = np.concatenate([self._noise, self._noise_rng.standard_normal(n)])
        self._native.set_noise(-1, self._noise)

    def step(self, max_iterations: int) -> _abi.TraceStatus:
        """Run up to max_iterations scheduler iterations on the device."""
        ne = self._native
        done = 0
        while True:
            it0 = self.iteration
            # one launch runs at most a ring's worth of iterations; its records are read
            # before the next launch can overwrite them
            ne.step(min(max_iterations - done, self.chunk_iterations), self.stream)
            st = ne.status(self.stream)[0]
            self.iteration = st.iterations
            done += st.iterations - it0
            self._read_records(st)
            if st.status != _abi.RS_RUNNING or done >= max_iterations:
                break
            # a launch that ran out of noise draws stops early, still running
            if self._noise_rng is not None and st.batches >= len(self._noise):
                self._extend_noise(len(self._noise))
        self._status = st
        self.iteration = st.iterations
        self.clock = st.clock
        self.kv_reserved = st.kv_reserved
        return st

    _n_read = 0

    def _read_records(self, st) -> None:
        if self.config.log_decisions and st.n_log > self._n_read:
            self._records.append(self._native.read_log(0, self._n_read, st.n_log - self._n_read))
            if self._record_order:
                R = self.trace.columns().num_relqueries
                self._orders.append(self._native.read_order(0, self._n_read, st.n_log - self._n_read, R))
                self._dpu_snaps.append(self._native.read_dpu(0, self._n_read, st.n_log - self._n_read, R))
            self._n_read = st.n_log

    def run(self) -> RunResult:
        t0 = time.perf_counter()
        while True:
            st = self.step(self.chunk_iterations)
            if st.status != _abi.RS_RUNNING:
                break
        wall = time.perf_counter() - t0
        self.result = self._collect(wall)
        if st.status != _abi.RS_OK:
            msgs = {
                _abi.RS_EABORT_LIMIT: f"iteration limit {self.config.iteration_limit} exceeded",
                _abi.RS_EABORT_IDLE: "engine idle with live relQueries and no future arrivals",
                _abi.RS_ECACHE_PINNED: "prefix cache cannot evict: all resident blocks pinned",
            }
            raise_for(st.status, msgs.get(st.status, f"device engine failed with status {st.status}"))
        return self.result

    def _collect(self, wall: float) -> RunResult:
        ne = self._native
        st = self._status
        c = self.trace.columns()
        arrival, fps, lpe, lde = ne.read_ledgers(0, c.num_relqueries)
        comp = ne.read_completion(0, c.num_requests)
        n_adm = int(st.admitted)

        def ledgers():  # admission order (arrival, rel_id), engine.py:211-213
            adm = np.lexsort((c.rel_id, c.arrival))[:n_adm]
            rid, av, fv, lv, dv = (c.rel_id.tolist(), arrival.tolist(), fps.tolist(), lpe.tolist(), lde.tolist())
            # NaN (x != x) -> None: the reference's unset timestamps
            return {rid[i]: TimestampLedger(av[i], None if fv[i] != fv[i] else fv[i],
                                            None if lv[i] != lv[i] else lv[i], None if dv[i] != dv[i] else dv[i])
                    for i in adm.tolist()}

        recs = (np.concatenate(self._records) if self._records
                else np.zeros(0, _abi.ITER_RECORD_DTYPE))
        log = _DecisionLog(recs if self.config.log_decisions else recs[:0])
        self._requests_state = None
        if self.trace.materialized:  # reference semantics: the run mutates the Request objects
            gen, pre, _, prio = self.requests_state
            k = 0
            g, p, pr = gen.tolist(), pre.tolist(), prio.tolist()
            for q in self.trace.entries:
                for r in q.requests:
                    r.generated, r.prefilled, r.priority = g[k], bool(p[k]), pr[k]
                    k += 1
        return RunResult(
            policy=self.policy, rate=self.trace.rate, seed=self.seed, ledgers=_LazyDict(ledgers),
            relquery_sizes=_LazyDict(lambda: dict(zip(c.rel_id.tolist(), np.diff(c.row_off).tolist()))),
            decision_log=log, iterations=int(st.iterations), sim_duration=float(st.clock),
            dpu_wall_s=self._phase_seconds(st, _DPU_PHASES), aba_wall_s=self._phase_seconds(st, _ABA_PHASES),
            cache_hit_tokens=int(st.cache_hit_tokens),
            cache_miss_tokens=int(st.cache_miss_tokens), completion_iteration=comp, records=recs,
            device_wall_s=wall, waiting_orders=self._waiting_orders(recs),
            **self._priority_records(),
        )

    def _priority_records(self) -> dict:
        if not self._record_order or self.policy in ("fcfs", "sp"):  # no DPU (engine.py:221-227)
            return {}
        c = self.trace.columns()
        adm = np.lexsort((c.rel_id, c.arrival))  # live_relqueries order (engine.py:211-213, 254)
        rid = c.rel_id[adm]
        recs, rngs = [], []
        for vals, flags, rng in self._dpu_snaps:
            v, f = vals[:, adm], flags[:, adm]
            for i in range(len(v)):
                live = (f[i] & _abi.SNAP_LIVE) != 0
                fi = f[i][live]
                recs.append(PriorityRecords(rid[live], v[i][live], (fi & _abi.SNAP_ESTIMATED) == 0,
                                            (fi & _abi.SNAP_OVERRIDE) != 0))
            for r in rng:
                rngs.append(((r.state_hi << 64) | r.state_lo, int(r.has_uint32), int(r.uinteger)))
        return {"priority_records": recs, "dpu_rng_states": rngs}

    def _waiting_orders(self, recs):
        if not self._record_order:
            return None
        rows = np.concatenate(self._orders) if self._orders else np.zeros((0, 0), np.int32)
        return [rows[i, : int(w)] for i, w in enumerate(recs["n_waiting"].tolist())]

    @property
    def requests_state(self):
        """(generated, prefilled, completion_iteration, priority) per request, trace order."""
        if getattr(self, "_requests_state", None) is None:
            self._requests_state = self._native.read_requests(0, self.trace.columns().num_requests)
        return self._requests_state

    def _phase_seconds(self, st, phases) -> float:
        """Device time of the given phases (clock64 cycles / SM clock)."""
        from . import _native

        khz = _native.device_clock_khz(self.device)
        return sum(int(st.phase_cycles[k]) for k in phases) / (khz * 1e3) if khz else 0.0

    def _admitted(self) -> np.ndarray:
        """Trace indices of the admitted relQueries in admission order (engine.py:211-213, 243-269)."""
        c = self.trace.columns()
        n_adm = int(self._status.admitted) if self._status is not None else 0
        return np.lexsort((c.rel_id, c.arrival))[:n_adm]

    @property
    def ledgers(self) -> dict:
        """relsim's ``Engine.ledgers`` (engine.py:207, 258-262) between steps: a TimestampLedger per
        admitted relQuery, in admission order, read from the device."""
        c = self.trace.columns()
        arrival, fps, lpe, lde = self._native.read_ledgers(0, c.num_relqueries)
        rid = c.rel_id
        nn = lambda x: None if x != x else float(x)  # noqa: E731  (NaN: unset)
        return {int(rid[i]): TimestampLedger(float(arrival[i]), nn(fps[i]), nn(lpe[i]), nn(lde[i]))
                for i in self._admitted().tolist()}

    @property
    def live_relqueries(self) -> dict:
        """relsim's ``Engine.live_relqueries`` (engine.py:208, 254, 362) between steps: the admitted
        relQueries with a request not yet done, in admission order (a relQuery without requests
        stays live, as in the reference)."""
        c = self.trace.columns()
        _, _, comp, _ = self._native.read_requests(0, c.num_requests)
        finished = comp >= 0
        sizes = np.diff(c.row_off)
        done_rows = np.zeros(c.num_relqueries, np.int64)
        rq_of_row = np.repeat(np.arange(c.num_relqueries), sizes)
        np.add.at(done_rows, rq_of_row[finished], 1)
        entries = self.trace.entries
        return {int(c.rel_id[i]): entries[i] for i in self._admitted().tolist()
                if sizes[i] == 0 or done_rows[i] < sizes[i]}

    @property
    def next_arrival(self) -> float | None:
        """relsim's ``Engine.next_arrival`` (engine.py:271-275): the arrival time of the next
        relQuery not admitted yet, or None."""
        c = self.trace.columns()
        n_adm = int(self._status.admitted) if self._status is not None else 0
        if n_adm >= c.num_relqueries:
            return None
        return float(c.arrival[np.lexsort((c.rel_id, c.arrival))[n_adm]])

    @property
    def kv_resident_tokens(self) -> int:
        """relsim's ``Engine.kv_resident_tokens`` (engine.py:365-367): tok + generated over the
        running requests."""
        rows = self.running_rows
        if not len(rows):
            return 0
        c = self.trace.columns()
        gen, _, _, _ = self._native.read_requests(0, c.num_requests)
        return int(c.tok[rows].sum() + gen[rows].sum())

    @property
    def dpu_wall(self) -> float:
        """Device time of the priority updates so far (relsim's ``dpu_wall``, engine.py:381-386)."""
        return self._phase_seconds(self._status, _DPU_PHASES) if self._status is not None else 0.0

    @property
    def aba_wall(self) -> float:
        """Device time of the waiting order, candidates and decisions so far (relsim's ``aba_wall``)."""
        return self._phase_seconds(self._status, _ABA_PHASES) if self._status is not None else 0.0

    @property
    def decision_log(self) -> list:
        """relsim's ``Engine.decision_log`` (engine.py:209, 419-433): the entries of the iterations
        run so far."""
        recs = np.concatenate(self._records) if self._records else np.zeros(0, _abi.ITER_RECORD_DTYPE)
        return list(_DecisionLog(recs)) if self.config.log_decisions else []

    def _row_objects(self):
        """Trace-order row k -> its Request object (reference objects, built on first use)."""
        if getattr(self, "_rows", None) is None:
            self._rows = [r for q in self.trace.entries for r in q.requests]
        return self._rows

    @property
    def running_rows(self) -> np.ndarray:
        """Trace-order request indices of the running list, in execution order (no objects)."""
        return self._native.read_running(0)

    @property
    def running(self) -> list:
        """relsim's ``Engine.running`` (engine.py:205): the prefilled, unfinished requests in
        execution order, as the trace's Request objects, read from the device between steps."""
        rows = self._row_objects()
        return [rows[k] for k in self.running_rows.tolist()]

    @property
    def waiting(self) -> list:
        """relsim's ``Engine.waiting`` (engine.py:160-176, 205, 277-281) between steps: one
        WaitingEntry per admitted relQuery with unprefilled requests, ordered by
        (priority, arrival, rel_id) -- the order of the last iteration's sort, whose head's
        prefilled rows have left ``pending``."""
        c = self.trace.columns()
        adm = np.lexsort((c.rel_id, c.arrival))  # admission order (engine.py:211-213)
        n_adm = int(self._status.admitted) if self._status is not None else 0
        _, pre, _, prio = self._native.read_requests(0, c.num_requests)
        entries = self.trace.entries
        out = []
        for ai, i in enumerate(adm[:n_adm].tolist()):
            lo, hi = int(c.row_off[i]), int(c.row_off[i + 1])
            n_pre = int(pre[lo:hi].sum())
            if n_pre < hi - lo:
                q = entries[i]
                e = WaitingEntry(q, ai)
                e.pending = q.requests[n_pre:]
                e._priority = float(prio[lo]) if hi > lo else 0.0
                out.append(e)
        out.sort(key=WaitingEntry.sort_key)
        return out

    def close(self):
        if getattr(self, "_native", None) is not None:
            self._native.close()
            self._native = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run(
    trace: ArrivalTrace,
    policy: str,
    world_model: LinearCostModel,
    config: EngineConfig | None = None,
    policy_model: LinearCostModel | None = None,
    seed: int = 0,
) -> RunResult:
    """Simulate serving the trace under the given policy to completion, on the GPU."""
    eng = Engine(trace, policy, world_model, config, policy_model, seed)
    try:
        return eng.run()
    finally:
        eng.close()
