"""Many independent traces in one engine (one CTA each): the config-4 building
block.  Every trace must match its own oracle run."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_multitrace_matches_oracle(oracle_mod):
    from paper_2601_11546_b200 import EngineConfig, TraceConfig, _abi, _marshal, generate_trace, world_preset
    from paper_2601_11546_b200._native import NativeEngine

    world = world_preset("llama-70b-like")
    cfg = EngineConfig()
    traces = [generate_trace(TraceConfig(num_relqueries=40, size_range=(1, s), rate=r, seed=i))
              for i, (s, r) in enumerate([(8, 4.0), (32, 1.0), (64, 0.5), (16, 2.0), (100, 0.25), (4, 8.0)])]
    ms = [_marshal.marshal_trace(t, cfg.block_size, "relserve", world) for t in traces]
    rngs = [_marshal.dpu_rng_state(i) for i in range(len(traces))]
    ne = NativeEngine([m.view for m in ms], _marshal.make_config(cfg, "relserve"), _marshal.make_model(world),
                      _marshal.make_model(world), rngs, 0, log_capacity=1 << 16)
    while True:
        ne.step(1 << 16)
        sts = ne.status()
        if all(s.status != _abi.RS_RUNNING for s in sts):
            break
    for i, (t, st) in enumerate(zip(traces, sts)):
        ref = oracle_mod.run(t, "relserve", world, cfg, None, i)
        assert st.status == 0 and ref.status == 0
        assert st.iterations == ref.iterations
        assert st.clock == ref.clock
        recs = ne.read_log(i, 0, st.n_log)
        for k in ("clock", "action", "kase", "head", "n_waiting", "batch_rq", "batch_first", "batch_n",
                  "kv_reserved"):
            assert np.array_equal(recs[k], ref.log[k]), (i, k)
        gen, pre, comp, prio = ne.read_requests(i, t.columns().num_requests)
        assert np.array_equal(comp, ref.completion_iter)
    ne.close()
