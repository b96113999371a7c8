"""Engine-creation timing breakdown (RS_TIMING=1 prints the native phases to stderr).

    RS_TIMING=1 python tools/create_timing.py CONFIG SHARDS [REPEATS]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_11546_b200 import _marshal  # noqa: E402
from paper_2601_11546_b200.engine import Engine, EngineConfig  # noqa: E402

cfg_id, shards = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
trace, world = bench.workload(cfg_id, 0)[:2]
trace.pin_memory()
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = _marshal.marshal_trace(trace, 16, "relserve", world, None)
    t1 = time.perf_counter()
    eng = Engine(trace, "relserve", world, EngineConfig(), device=0, shards=shards)
    t2 = time.perf_counter()
    eng.step(1)
    t3 = time.perf_counter()
    eng.close()
    t4 = time.perf_counter()
    print(f"rep {r}: marshal {1e3*(t1-t0):.2f} ms, Engine() {1e3*(t2-t1):.2f} ms, step(1) {1e3*(t3-t2):.2f} ms, "
          f"close {1e3*(t4-t3):.2f} ms", flush=True)
