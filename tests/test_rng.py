"""numpy PCG64 / Generator.choice(replace=False) replay (oracle side; the
device replay is checked in test_gpu_units.py)."""

import numpy as np
import pytest

from paper_2601_11546_b200 import _abi


@pytest.mark.parametrize("seed", [0, 1, 7, 12345])
def test_choice_sequence_matches_numpy(seed, oracle_mod):
    g = np.random.default_rng(np.random.SeedSequence([seed, 0xD9]))
    st = _abi.Pcg64State.from_numpy(g.bit_generator.state)
    rs = np.random.default_rng(seed)
    for _ in range(300):
        n = int(rs.integers(2, 3000))
        k = int(min(n - 1, rs.integers(1, 12)))
        want = g.choice(n, size=k, replace=False)
        got = oracle_mod.choice(st, n, k)
        assert got.tolist() == want.tolist()
    assert st.to_numpy()["state"] == g.bit_generator.state["state"]
    assert st.to_numpy()["has_uint32"] == g.bit_generator.state["has_uint32"]


def test_next32_buffering(oracle_mod):
    g = np.random.Generator(np.random.PCG64(5))
    st = _abi.Pcg64State.from_numpy(g.bit_generator.state)
    L = oracle_mod.lib()
    import ctypes

    want = g.integers(0, 2**32, size=9, dtype=np.uint64, endpoint=False)
    # integers(0, 2**32) draws one next32 per value (masked path uses full 32 bits)
    got = [L.or_next32(ctypes.byref(st)) for _ in range(9)]
    assert got == want.tolist()
