"""B200-native RelServe scheduling hot path (drop-in for relsim's engine API).

The public names mirror `relsim` (pkg/src/relsim/__init__.py:3-25) for the
scheduling path: state types and traces, the iteration cost model, the
scheduler constraints / priority types, and `run`/`Engine`, whose loop runs
on the GPU.
"""

from .cost_model import (
    WORLD_PRESETS,
    LinearCostModel,
    load_model,
    predict_decode,
    predict_prefill,
    save_model,
    world_preset,
)
from .engine import (
    POLICIES,
    DecisionLogEntry,
    Engine,
    EngineConfig,
    RunResult,
    SimulationAborted,
    TimestampLedger,
    run,
)
from .priority import (
    CacheMissRatio,
    DynamicPriorityUpdater,
    InfeasibleRequestError,
    PriorityRecord,
    RemainderItem,
    SchedulerConstraints,
    apply_starvation_override,
    pem,
    pem_batch,
    remainder_items,
    sample_cache_miss_ratio,
    static_relquery_prio,
    static_req_prio,
    utok_approx,
)
from .report import SummaryTable, decompose, summarize
from .workload import (
    OUTPUT_LIMITS,
    ArrivalTrace,
    QueryType,
    RelQuery,
    Request,
    TraceColumns,
    TraceConfig,
    generate_heavy_tail_trace,
    generate_trace,
    load_trace,
    save_trace,
)

__all__ = [
    "apply_starvation_override", "ArrivalTrace", "CacheMissRatio", "DecisionLogEntry", "DynamicPriorityUpdater", "decompose", "Engine", "EngineConfig", "InfeasibleRequestError",
    "LinearCostModel", "OUTPUT_LIMITS", "POLICIES", "PriorityRecord", "QueryType", "RelQuery",
    "RemainderItem", "Request", "RunResult", "SchedulerConstraints", "SimulationAborted",
    "TimestampLedger", "TraceColumns", "TraceConfig", "WORLD_PRESETS", "generate_heavy_tail_trace",
    "generate_trace", "load_model", "load_trace", "pem", "pem_batch", "predict_decode", "predict_prefill",
    "remainder_items", "run", "sample_cache_miss_ratio", "save_model", "save_trace", "static_relquery_prio", "static_req_prio",
    "summarize", "SummaryTable", "utok_approx", "world_preset",
]
