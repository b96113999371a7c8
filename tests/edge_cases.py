"""Hand-built edge-case traces shared by the reference-side golden generator
(tests/golden/make_edge_golden.py) and the device test (tests/test_gpu_edge_cases.py)."""

CAP = (2000, 8, 400)  # (cap, max_num_seqs, max_num_batched_tokens)

CASES = {
    # no relQuery at all: the loop never runs (engine.py:375)
    "empty": {"constraints": CAP, "rq": []},
    # one request
    "single": {"constraints": CAP, "rq": [(7, 0.25, 5, [(33, 5)])]},
    # a relQuery without requests never retires: the engine idles with it live (engine.py:441-445)
    "zero_size": {"constraints": CAP, "rq": [(0, 0.0, 5, []), (1, 0.1, 5, [(20, 3)])]},
    # tok + output_limit == cap: feasible, the whole KV budget (engine.py:235-239)
    "kv_exact_cap": {"constraints": CAP, "rq": [(3, 0.0, 100, [(1900, 100), (1900, 50)])]},
    # tok + output_limit == cap + 1: infeasible up front
    "kv_over_cap": {"constraints": CAP, "rq": [(3, 0.0, 100, [(1901, 100)])]},
    # a row longer than max_num_batched_tokens prefills alone (arranger.py:99-110, `taken` guard)
    "row_over_mnbt": {"constraints": CAP, "rq": [(5, 0.0, 10, [(500, 4), (30, 10), (450, 2)])]},
    # ragged: sizes 1..9 arriving together, more rows than max_num_seqs
    "ragged_burst": {"constraints": CAP,
                     "rq": [(10 + i, 0.0, 10, [(17 + 13 * j % 90, 1 + j % 10) for j in range(i + 1)])
                            for i in range(9)]},
    # identical arrival times and sizes: order falls to rel_id (engine.py:175-176, 211-213)
    "ties": {"constraints": CAP, "rq": [(40 - i, 0.5, 5, [(64, 5), (64, 5)]) for i in range(6)]},
}


def build(spec, ArrivalTrace, RelQuery, Request):
    """The trace of one case; token ids are distinct per request (no shared prefix)."""
    entries = []
    for rel_id, arrival, ol, rows in spec["rq"]:
        reqs = [Request(rel_id, j, [rel_id * 100000 + j * 10000 + t for t in range(tok)], ol, out, arrival)
                for j, (tok, out) in enumerate(rows)]
        entries.append(RelQuery(rel_id, reqs, ol, arrival))
    return ArrivalTrace(entries, 1.0, 0)
