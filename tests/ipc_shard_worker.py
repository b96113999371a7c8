"""Helper for tests/test_gpu_sharded.py::test_two_process_shards_over_ipc: one
shard of a sharded pool per process (mailboxes exchanged as CUDA IPC handles
over a gloo group), all on GPU 0 -- or, with RS_IPC_DEVICE_PER_RANK=1, rank r on
GPU r (tests/test_gpu_multigpu.py: the NVLink peer-memory path).  Not collected
by pytest (no test_ prefix)."""

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(rank: int, world: int, port: int, out_path: str):
    import numpy as np
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_11546_b200 import EngineConfig, TraceConfig, generate_trace, sharded, world_preset
    from paper_2601_11546_b200.engine import Engine, SimulationAborted

    n_rq = int(os.environ.get("RS_IPC_RELQUERIES", "40"))
    trace = generate_trace(TraceConfig(num_relqueries=n_rq, size_range=(1, 60), rate=4.0, seed=9))
    cfg = EngineConfig(iteration_limit=int(os.environ.get("RS_IPC_ITERS", "40")))
    device = rank if os.environ.get("RS_IPC_DEVICE_PER_RANK") == "1" else 0
    eng = Engine(trace, "relserve", world_preset("opt-13b-like"), cfg, device=device, shards=world, shard_rank=rank)
    sharded.connect(eng)
    try:
        res = eng.run()
    except SimulationAborted:
        res = eng.result
    np.save(out_path, res.records)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
