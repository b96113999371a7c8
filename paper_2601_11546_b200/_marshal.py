"""Trace/config marshalling into the C-ABI structs (host side of the boundary).

Builds the column arrays an `rs_trace_view` points at, including the
prefix-cache structure the device model needs: for every relQuery the number
of leading whole blocks shared by all its rows (``chain_blocks``).  For
count-keyed traces (generate_trace / load_trace) that is prefix_len //
block_size by construction.  For traces built from
explicit token lists the static block trie is computed here and checked to
be a forest of per-relQuery chains with private per-row tails; anything else
is rejected loudly (RS_EUNSUPPORTED) -- there is no CPU fallback.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _abi
from .workload import ArrivalTrace


class UnsupportedTraceError(NotImplementedError):
    """The trace's prefix structure is outside the device prefix-cache model."""


@dataclass
class StaticTrie:
    path_off: np.ndarray    # int64[N+1]
    path_node: np.ndarray   # int32[sum nblocks]
    node_parent: np.ndarray  # int32[n_nodes]


def static_trie(trace: ArrivalTrace, block_size: int) -> StaticTrie:
    """Static trie of all whole blocks of all requests (explicit tokens)."""
    node_of: dict = {}
    parents: list[int] = []
    offs = [0]
    nodes: list[int] = []
    B = block_size
    for q in trace.entries:
        for r in q.requests:
            toks = r.tokens
            parent = -1
            for j in range(len(toks) // B):
                key = (parent, tuple(toks[j * B:(j + 1) * B]))
                nid = node_of.get(key)
                if nid is None:
                    nid = len(parents)
                    node_of[key] = nid
                    parents.append(parent)
                nodes.append(nid)
                parent = nid
            offs.append(len(nodes))
    return StaticTrie(np.asarray(offs, np.int64), np.asarray(nodes, np.int32),
                      np.asarray(parents, np.int32))


def chain_blocks_from_trie(trace: ArrivalTrace, trie: StaticTrie) -> np.ndarray:
    """Per-relQuery shared chain length; raises if the trie is not chain+tails."""
    c = trace.columns()
    R = c.num_relqueries
    n_nodes = trie.node_parent.shape[0]
    uses = np.zeros(n_nodes, np.int64)
    owner = np.full(n_nodes, -1, np.int64)
    np.add.at(uses, trie.path_node, 1)
    chain = np.zeros(R, np.int32)
    off = c.row_off
    po = trie.path_off
    for q in range(R):
        rows = range(off[q], off[q + 1])
        paths = [trie.path_node[po[r]:po[r + 1]] for r in rows]
        for p in paths:
            for nid in p.tolist():
                if owner[nid] == -1:
                    owner[nid] = q
                elif owner[nid] != q:
                    raise UnsupportedTraceError(
                        f"relQueries {int(c.rel_id[owner[nid]])} and {int(c.rel_id[q])} share a "
                        "prefix block; the device prefix-cache model needs per-relQuery forests")
        if len(paths) >= 2:
            lcp = min(len(p) for p in paths)
            for p in paths[1:]:
                neq = np.nonzero(p[:lcp] != paths[0][:lcp])[0]
                if neq.size:
                    lcp = int(neq[0])
            chain[q] = lcp
        size = len(paths)
        for p in paths:
            P = int(chain[q])
            if P and np.any(uses[p[:P]] != size):
                raise UnsupportedTraceError("shared chain is not shared by every row")
            if np.any(uses[p[P:]] != 1):
                raise UnsupportedTraceError(
                    f"relQuery {int(c.rel_id[q])}: rows share blocks beyond the common prefix")
    return chain


@dataclass
class Marshalled:
    view: _abi.TraceView
    arrays: dict
    trie: StaticTrie | None


def marshal_trace(trace: ArrivalTrace, block_size: int, policy: str, policy_model, sp_fns=None,
                  need_trie: bool = False, check_forest: bool = True) -> Marshalled:
    """Column arrays + rs_trace_view for one trace (arrays kept alive in the result)."""
    c = trace.columns()
    explicit = c.token_seed is None
    if trace.materialized:
        for q in trace.entries:
            for r in q.requests:
                if r.output_limit != q.output_limit:
                    raise UnsupportedTraceError(
                        f"request {q.rel_id}/{r.req_id}: output_limit differs from its relQuery's")
    trie = None
    if explicit:
        trie = static_trie(trace, block_size)
        chain = chain_blocks_from_trie(trace, trie) if check_forest else np.zeros(c.num_relqueries, np.int32)
    else:
        chain = (c.prefix_len // block_size).astype(np.int32)
        if need_trie:
            trie = None  # oracle synthesises the same structure from chain_blocks
    static_prio = None
    if policy == "sp":
        static_prio = _static_priorities(trace, policy_model, sp_fns)
    arrays = {
        "rel_id": np.ascontiguousarray(c.rel_id, np.int64),
        "arrival": np.ascontiguousarray(c.arrival, np.float64),
        "output_limit": np.ascontiguousarray(c.output_limit, np.int32),
        "row_off": np.ascontiguousarray(c.row_off, np.int64),
        "tok": np.ascontiguousarray(c.tok, np.int32),
        "out": np.ascontiguousarray(c.out, np.int32),
        "chain_blocks": np.ascontiguousarray(chain, np.int32),
        "static_prio": None if static_prio is None else np.ascontiguousarray(static_prio, np.float64),
    }
    view = _abi.TraceView(
        c.num_relqueries, c.num_requests,
        *(_abi.ptr(arrays[k]) for k in ("rel_id", "arrival", "output_limit", "row_off", "tok",
                                         "out", "chain_blocks", "static_prio")),
    )
    return Marshalled(view, arrays, trie)


def _static_priorities(trace: ArrivalTrace, model, sp_fns) -> np.ndarray:
    """static_relquery_prio per relQuery (engine.py:255-264, priority.py:221-235).

    The reference sums with the builtin ``sum`` (Neumaier-compensated since
    CPython 3.12, plain left-to-right before), so this does too: the static
    priorities are bit-identical under the running interpreter.  Default
    mappings are alpha_p*tok and alpha_d*ol of the policy model
    (engine.py:259-261).  Any sign is allowed (the device orders priorities by
    an order-preserving key, engine_state.cuh okey()).
    """
    c = trace.columns()
    out = np.zeros(c.num_relqueries, np.float64)
    off = c.row_off.tolist()
    if sp_fns is None:
        ol = np.repeat(c.output_limit.astype(np.float64), np.diff(c.row_off))
        vals = (model.alpha_p * c.tok.astype(np.float64) + model.alpha_d * ol).tolist()
        for q in range(c.num_relqueries):
            out[q] = sum(vals[off[q]:off[q + 1]])  # the running interpreter's sum, as the reference's
        return out
    l1, l2 = sp_fns
    for q, rq in enumerate(trace.entries):
        out[q] = float(sum(l1(r.tok) + l2(r.output_limit) for r in rq.requests))
    return out


def make_config(cfg, policy: str, record_order: bool = False) -> _abi.Config:
    cons = cfg.constraints
    return _abi.Config(
        record_order=int(bool(record_order)),
        cap=cons.cap, max_num_seqs=cons.max_num_seqs,
        max_num_batched_tokens=cons.max_num_batched_tokens,
        sample_size=cfg.sample_size, tau=float(cfg.tau), noise_sigma=float(cfg.noise_sigma),
        block_size=cfg.block_size, capacity_blocks=cfg.capacity_blocks,
        iteration_limit=min(int(cfg.iteration_limit), 2**62) if not math.isinf(cfg.iteration_limit) else 2**62,
        log_decisions=int(bool(cfg.log_decisions)), policy=_abi.POLICY_IDS[policy],
    )


def make_model(m) -> _abi.CostModel:
    return _abi.CostModel(m.alpha_p, m.beta_p, m.alpha_d, m.beta_d)


def dpu_rng_state(seed: int) -> _abi.Pcg64State:
    """DPU generator start state: default_rng(SeedSequence([seed, 0xD9])) (engine.py:224)."""
    g = np.random.default_rng(np.random.SeedSequence([seed, 0xD9]))
    return _abi.Pcg64State.from_numpy(g.bit_generator.state)
