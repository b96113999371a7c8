"""Workloads and run fingerprints shared by tests/test_gpu_fullscale.py and
tests/golden/make_fullscale.py (BASELINE configs 2 and 3 at full size)."""

import hashlib

import numpy as np

_NAN = np.int64(0x7FF8000000000000)


def _config2():
    from paper_2601_11546_b200 import EngineConfig, TraceConfig, generate_trace, world_preset

    t = generate_trace(TraceConfig(num_relqueries=1000, size_range=(1000, 1000), rate=1e6, seed=0))
    return t, world_preset("opt-13b-like"), EngineConfig()


def _config3():
    from paper_2601_11546_b200 import EngineConfig, generate_heavy_tail_trace, world_preset

    t = generate_heavy_tail_trace(num_relqueries=5000, size_range=(1, 399), rate=1e6, seed=0)
    return t, world_preset("llama-70b-like"), EngineConfig()


def _config5():
    from paper_2601_11546_b200 import EngineConfig, generate_heavy_tail_trace, world_preset

    t = generate_heavy_tail_trace(num_relqueries=40000, size_range=(1, 399), rate=1e6, seed=0)
    return t, world_preset("llama-70b-like"), EngineConfig()


WORKLOADS = {"config2": _config2, "config3": _config3, "config5": _config5}

#: complete runs fingerprinted: name -> (workload, policy)
RUNS = {"config2": ("config2", "relserve"), "config3": ("config3", "relserve"),
        "config3_fcfs": ("config3", "fcfs"), "config3_sp": ("config3", "sp"),
        "config3_pp": ("config3", "relserve-pp"), "config3_dp": ("config3", "relserve-dp"),
        "config2_fcfs": ("config2", "fcfs"), "config2_sp": ("config2", "sp"),
        "config2_pp": ("config2", "relserve-pp"), "config2_dp": ("config2", "relserve-dp")}

#: windowed runs at full size: name -> (workload, policy, iterations).  Config 5 (one pool of
#: 8e6 requests) runs for hours on one core, so its first WINDOW iterations are fingerprinted
#: (first sight of all 40,000 relQueries included) and the device compared over the same window
WINDOWS = {"config5_window": ("config5", "relserve", 3000)}

#: decision-record fields compared (rs_iter_record; the oracle's log has the same names)
FIELDS = ("iteration", "clock", "m_plus", "m_minus", "delta_plus", "delta_minus", "delta_total", "kv_reserved",
          "action", "kase", "head", "n_waiting", "batch_rq", "batch_first", "batch_n", "n_reestimated")


def _canon(a: np.ndarray) -> bytes:
    a = np.asarray(a)
    if a.dtype.kind == "f":
        b = a.astype("<f8").view("<i8").copy()
        b[np.isnan(a)] = _NAN
        return b.tobytes()
    return a.astype("<i8").tobytes()


def fingerprint(records: np.ndarray, completion: np.ndarray) -> dict:
    fp = {f"sha256_{k}": hashlib.sha256(_canon(records[k])).hexdigest() for k in FIELDS}
    fp["sha256_completion"] = hashlib.sha256(_canon(completion)).hexdigest()
    fp["records"] = int(len(records))
    return fp
