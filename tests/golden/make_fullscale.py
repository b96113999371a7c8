"""Fingerprints of complete runs at BASELINE's full sizes (configs 2 and 3,
10^6 requests each) computed by the CPU oracle -- the C restatement that
tests/golden/*.json.gz pin to the real reference -- for
tests/test_gpu_fullscale.py to compare the device's complete runs against bit
for bit.  The Python reference would need hours per run here (3.8 iters/s);
the oracle takes about a minute.  Run from the repo root:

    python tests/golden/make_fullscale.py [run names]

writes tests/golden/fullscale.json: per config the iteration count, the final
clock and cache counters (exact, as repr / ints) and a SHA-256 per decision-record
field and of the per-request completion iterations (canonical little-endian int64
/ float64 bits, every NaN as one bit pattern).
"""

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from fullscale_util import RUNS, WINDOWS, WORKLOADS, fingerprint  # noqa: E402


def main():
    from oracle import oracle

    oracle.build()
    path = Path(__file__).parent / "fullscale.json"
    out = json.loads(path.read_text()) if path.exists() else {"numpy": np.__version__, "configs": {}}
    only = set(sys.argv[1:])
    for name, (wl, policy) in RUNS.items():
        if only and name not in only:
            continue
        trace, world, cfg = WORKLOADS[wl]()
        t0 = time.perf_counter()
        r = oracle.run(trace, policy, world, cfg, None, 0)
        wall = time.perf_counter() - t0
        assert r.status == 0, r.message
        fp = fingerprint(r.log, r.completion_iter)
        fp.update({"iterations": int(r.iterations), "clock": repr(float(r.clock)),
                   "cache_hit_tokens": int(r.cache_hit_tokens), "cache_miss_tokens": int(r.cache_miss_tokens),
                   "oracle_wall_s": round(wall, 1), "workload": wl, "policy": policy})
        out["configs"][name] = fp
        print(name, r.iterations, f"{wall:.1f} s", flush=True)
        path.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    from dataclasses import replace

    for name, (wl, policy, n) in WINDOWS.items():
        if only and name not in only:
            continue
        trace, world, cfg = WORKLOADS[wl]()
        t0 = time.perf_counter()
        r = oracle.run(trace, policy, world, replace(cfg, iteration_limit=n), None, 0)
        wall = time.perf_counter() - t0
        assert r.status == 3 and r.iterations == n, (r.status, r.iterations, r.message)  # SimulationAborted at n
        fp = fingerprint(r.log, r.completion_iter)
        fp.update({"iterations": int(r.iterations), "clock": repr(float(r.clock)),
                   "cache_hit_tokens": int(r.cache_hit_tokens), "cache_miss_tokens": int(r.cache_miss_tokens),
                   "kv_reserved": int(r.kv_reserved), "oracle_wall_s": round(wall, 1), "workload": wl,
                   "policy": policy, "window": n})
        out["windows"] = out.get("windows", {})
        out["windows"][name] = fp
        print(name, r.iterations, f"{wall:.1f} s", flush=True)
        path.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
