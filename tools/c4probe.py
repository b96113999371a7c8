import sys, time, json
sys.path.insert(0, '.')
import torch
import bench
from paper_2601_11546_b200 import EngineConfig, TraceConfig, generate_trace, world_preset, _marshal, _abi
from paper_2601_11546_b200._native import NativeEngine
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
cells = bench.config4_cells(); mine = list(range(0, len(cells), 8))[:128]
cfg = EngineConfig(); c_cfg = _marshal.make_config(cfg, "relserve")
by = {}
for ci in mine:
    m, r, s = cells[ci]
    by.setdefault(m, []).append((ci, generate_trace(TraceConfig(num_relqueries=100, size_range=(1, s), rate=r, seed=ci)).pin_memory()))
G = int(sys.argv[1]) if len(sys.argv) > 1 else 16
groups = []
for m, it in by.items():
    it.sort(key=lambda x: -x[1].columns().num_requests)
    groups += [(m, it[k:k+G]) for k in range(0, len(it), G)]
groups.sort(key=lambda g: -g[1][0][1].columns().num_requests)
streams = [torch.cuda.Stream(dev) for _ in groups]
print("stream flags nonblocking?", [s.cuda_stream for s in streams][:2])
for rep in range(4):
    t0 = time.perf_counter(); marks = []
    engs = []
    for (m, it), st in zip(groups, streams):
        w = world_preset(m)
        a = time.perf_counter()
        ms = [_marshal.marshal_trace(t, 16, "relserve", w) for _, t in it]
        rngs = [_marshal.dpu_rng_state(ci) for ci, _ in it]
        b = time.perf_counter()
        ne = NativeEngine([x.view for x in ms], c_cfg, _marshal.make_model(w), _marshal.make_model(w), rngs, 0, log_capacity=0)
        c = time.perf_counter()
        ne.step(1 << 30, st)
        d = time.perf_counter()
        marks.append((round(1e3*(b-a),2), round(1e3*(c-b),2), round(1e3*(d-c),2)))
        engs.append((ne, ms))
    t1 = time.perf_counter()
    waits = []
    for (ne, ms), st in zip(engs, streams):
        a = time.perf_counter(); ne.status(st); b = time.perf_counter()
        R = sum(x.view.num_relqueries for x in ms); N = sum(x.view.num_requests for x in ms)
        ne.read_results(R, N, st); c = time.perf_counter()
        waits.append((round(1e3*(b-t0),2), round(1e3*(c-b),2)))
    t2 = time.perf_counter()
    for ne, _ in engs: ne.close()
    print(rep, "build", round(1e3*(t1-t0),2), "total", round(1e3*(t2-t0),2), marks, waits)
