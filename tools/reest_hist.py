"""Histogram of re-estimated relQueries per iteration (the pipelined update's fast path holds
kSmallEst = 32 of them and kMaxJobs = 64 PEM segments; larger iterations update in place).

    python tools/reest_hist.py CONFIG [ITERATIONS]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2601_11546_b200.engine import Engine  # noqa: E402

trace, world, cfg, _ = bench.workload(sys.argv[1], 0)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3255
e = Engine(trace, "relserve", world, cfg, device=0)
e.step(n)
r = np.concatenate(e._records)
x = r["n_reestimated"][5:]
print(f"config {sys.argv[1]}: {len(x)} iterations, mean {x.mean():.2f}, > 32: {np.mean(x > 32):.3f}, "
      f"> 48: {np.mean(x > 48):.3f}, > 64: {np.mean(x > 64):.3f}, max {x.max()}")
print("percentiles 50/90/99:", np.percentile(x, [50, 90, 99]))
e.close()
