"""Golden records of relsim's DynamicPriorityUpdater (priority.py:238-339) over the
scripted update sequences of tests/dpu_scenario.py (test infrastructure; runs in
the build container where the reference is mounted):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_dpu_golden.py
"""

from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
from relsim.cost_model import LinearCostModel  # noqa: E402
from relsim.priority import DynamicPriorityUpdater, SchedulerConstraints  # noqa: E402
from relsim.workload import RelQuery, Request  # noqa: E402

import dpu_scenario  # noqa: E402

MODEL = (0.001, 0.02, 0.0002, 0.015)
CONS = (2000, 16, 400)


def main():
    for name, (seed, n_rq, iters, tau, k) in dpu_scenario.SCENARIOS.items():
        rqs = dpu_scenario.build(seed, n_rq, Request, RelQuery)
        cache = dpu_scenario.StubCache()
        dpu = DynamicPriorityUpdater(SchedulerConstraints(*CONS), LinearCostModel(*MODEL), cache, sample_size=k,
                                     tau=tau, rng=np.random.default_rng(np.random.SeedSequence([seed, 0xD9])))
        recs, states = dpu_scenario.drive(dpu, cache, rqs, iters, seed)
        doc = {"name": name, "model": MODEL, "constraints": CONS, "numpy": np.__version__,
               "records": [[[rid, v.hex(), ic, ru, ov] for rid, v, ic, ru, ov in it] for it in recs],
               "rng": [[str(s), h, u] for s, h, u in states]}
        path = ROOT / "tests" / "golden" / "dpu_api" / f"{name}.json.gz"
        with gzip.open(path, "wt") as f:
            json.dump(doc, f)
        n = sum(len(it) for it in recs)
        est = sum(1 for it in recs for r in it if not r[3])
        print(f"{name}: {iters} updates, {n} records ({est} estimated) -> {path.name}")


if __name__ == "__main__":
    main()
