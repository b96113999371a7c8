"""Count discarded speculations of the pipelined update over the common-kernel sweep cases
(RS_LIB=scratch/lib_misspec.so, built with -DRS_COUNT_MISSPEC=1)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
from paper_2601_11546_b200 import SchedulerConstraints, TraceConfig, generate_trace, world_preset  # noqa: E402
from paper_2601_11546_b200.engine import Engine, EngineConfig  # noqa: E402
import test_gpu_sweep as sw  # noqa: E402

tot = iters = 0
for i in range(60):
    tc, cons, kw, policy, model, seed, _ = sw._common_case(i)
    cfg = EngineConfig(constraints=SchedulerConstraints(*cons), iteration_limit=20_000, **kw)
    try:
        e = Engine(generate_trace(TraceConfig(**tc)), policy, world_preset(model), cfg, None, seed, device=0)
        try:
            e.run()
        except Exception:
            pass
        st = e._status
        tot += int(st.phase_cycles[20])
        iters += int(st.iterations)
        e.close()
    except Exception as ex:  # noqa: BLE001
        print(i, "skipped:", ex)
print({"discarded_speculations": tot, "iterations": iters})
