#!/usr/bin/env python
"""Benchmark: scheduler iterations/s at 10^6 pending requests (BASELINE.json).

Workload (config 2 of BASELINE.json): 1,000 relQueries x 1,000 rows
(10^6 requests, all arriving within ~1 ms), opt-13b-like cost model (the
only 13B preset; "Llama-2-13B" maps to it), EngineConfig() defaults, policy
relserve, engine seed 0.  A *step* is one launch of the persistent scheduler
kernel that advances the trace by `--iters-per-step` scheduler iterations.
Iterations [0, 5) run first (admission and the first-sight DPU pass, as in
SURVEY 8d); then W warm-up steps, then K timed steps, each bracketed by CUDA
events on the launching stream, with a 256 MiB L2 flush between steps
(outside the events).  The timed window is iterations [5 + W*I, 5 + (W+K)*I),
printed as config.window_start/end_iteration -- the same window the reference
arm times.  `value` = iterations / summed step time.

`e2e` runs iterations [0, window end) through the public API (`Engine` over
host arrays): trace upload, every step's launch, status and decision-record
readback, and the final ledger/request readback are inside the wall-clock
timed region.

`--impl reference` times the CPU restatement of the reference engine
(oracle/, single-threaded like the reference) on the same trace and window.

Multi-GPU (torchrun, N ranks): every rank runs an independent config-2 trace
(seed = rank); value = all ranks' iterations / max-over-ranks time (weak
scaling; a single trace's iterations are serially dependent).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sched iters/sec @1M pending reqs"
PHASES = ("admit", "dpu_other", "order", "decision", "execute", "dpu_setup", "dpu_rng", "dpu_summaries",
          "dpu_pem", "fp_evict_post", "prefill_post", "cand_decode", "cand_prefill", "fp_scan", "fp_stage",
          "dpu_ratio", "p16", "p17", "p18", "p19", "p20", "p21", "p22")
WINDOW_START = 5
#: per-config ncu numbers of the dominant kernel from the committed `ncu --set full` capture
#: (dram__bytes_read.sum + dram__bytes_write.sum per launch; tools/ncu_traffic.py writes it)
TRAFFIC_FILE = ROOT / "profiles" / "traffic.json"
L2_NOTE = ("GPU arm: a 256 MiB buffer is written between timed steps (outside the events); "
           "CPU arm: not applicable")


def traffic(cfg_id: str, iters_per_step: int):
    """ncu DRAM bytes per launch of the bench's kernel for this config, scaled to this launch
    size, with the capture it comes from (None if no capture of this config is committed)."""
    try:
        d = json.loads(TRAFFIC_FILE.read_text()).get(f"config{cfg_id}")
    except (OSError, ValueError):
        d = None
    if not d:
        return None, None
    per_iter = d["dram_bytes_per_launch"] / d["iters_per_launch"]
    return per_iter * iters_per_step, d


def window_stats(recs, comp, c, lo: int, hi: int) -> dict:
    """The workload at the timed window [lo, hi) from a run's decision records (all
    iterations from 0) and per-request completion iterations: requests waiting at lo, and the
    mean live requests / relQueries over the window (B_iter = 6 N_live + 56 R_live)."""
    it = recs["iteration"]
    clock_lo = float(recs["clock"][np.searchsorted(it, lo)]) if len(it) and lo <= it[-1] else math.inf
    sizes = np.diff(c.row_off)
    adm_rq = c.arrival <= clock_lo  # admitted by iteration lo (engine.py:243-249)
    n_adm = int(sizes[adm_rq].sum())
    pf = (recs["action"] == 0) & (it < lo)
    pending = n_adm - int(recs["batch_n"][pf].sum())
    ts = np.arange(lo, hi)
    done = np.sort(comp[comp >= 0])
    n_live = n_adm - np.searchsorted(done, ts, side="left")  # rows done before t are not live at t
    rq_of = np.repeat(np.arange(c.num_relqueries), sizes)
    last = np.full(c.num_relqueries, -1, np.int64)
    np.maximum.at(last, rq_of, np.where(comp < 0, np.iinfo(np.int64).max // 2, comp))
    rq_done = np.sort(last[adm_rq & (sizes > 0)])
    r_live = int((adm_rq & (sizes > 0)).sum()) - np.searchsorted(rq_done, ts, side="left")
    return {"pending_requests_start": int(pending), "live_requests_mean": float(n_live.mean()),
            "live_relqueries_mean": float(r_live.mean())}


def b_iter(ws: dict) -> float:
    """SURVEY 8d's declared algorithmic bytes per iteration: 6 N_live + 56 R_live."""
    return 6.0 * ws["live_requests_mean"] + 56.0 * ws["live_relqueries_mean"]


def config_dict(wname: str, I: int, lo: int, hi: int, ws: dict) -> dict:
    """The `config` of both arms' lines (identical keys and values for the same run shape)."""
    return {"workload": wname, "iters_per_step": I, "window_start_iteration": lo, "window_end_iteration": hi,
            "pending_requests_start": ws["pending_requests_start"], "l2": L2_NOTE}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--iters-per-step", type=int, default=250)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["2", "3", "4", "5"], default="2")
    ap.add_argument("--shards", type=int, default=None,
                    help="config 5 on one GPU: shards as CTAs of one launch (default 8); under torchrun "
                         "every rank is one shard")
    ap.add_argument("--traces-per-gpu", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=6000)
    return ap.parse_args()


def workload(cfg_id: str, seed: int):
    from paper_2601_11546_b200 import (EngineConfig, TraceConfig, generate_heavy_tail_trace,
                                       generate_trace, world_preset)

    if cfg_id == "2":
        trace = generate_trace(TraceConfig(num_relqueries=1000, size_range=(1000, 1000), rate=1e6, seed=seed))
        world = world_preset("opt-13b-like")
        name = "config2: 1000 relQ x 1000 rows, opt-13b-like (Llama-2-13B), relserve"
    elif cfg_id == "3":
        trace = generate_heavy_tail_trace(num_relqueries=5000, size_range=(1, 399), rate=1e6, seed=seed)
        world = world_preset("llama-70b-like")
        name = "config3: 5000 relQ x U[1,399] heavy-tailed outputs, llama-70b-like (Llama-2-70B), relserve"
    else:
        trace = generate_heavy_tail_trace(num_relqueries=40000, size_range=(1, 399), rate=1e6, seed=seed)
        world = world_preset("llama-70b-like")
        name = ("config5: one pool of 40000 relQ x U[1,399] (8e6 requests) heavy-tailed outputs, "
                "llama-70b-like (Llama-2-70B), relserve, relQueries sharded round-robin")
    return trace, world, EngineConfig(), name


def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # tests only: every rank on one device (the multi-rank path on a one-GPU box; NCCL refuses
    # two ranks per GPU, so the plumbing goes over gloo)
    shared = os.environ.get("RS_BENCH_DEVICE")
    if shared is not None:
        local = int(shared)
    if ws > 1:
        import torch.distributed as dist

        backend = "nccl" if args.impl == "ours" and shared is None else "gloo"
        if backend == "nccl":
            import torch

            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return ws, rank, local


def max_over_ranks(x: float, ws: int, device=None) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, ws: int, device=None) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region.

    NVML polled from a thread every ~1 ms (the timed regions here last tens of
    ms, shorter than nvidia-smi's sampling period); nvidia-smi as the fallback."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.thread = None
        self.sm, self.mx, self.reasons = [], None, set()

    def _poll(self):
        import pynvml as N

        h = N.nvmlDeviceGetHandleByIndex(self.index)
        self.mx = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
        flags = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                 "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        while not self.stop:
            self.sm.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
            r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.reasons.update(k for k, f in flags.items() if r & f)
            time.sleep(0.001)

    def __enter__(self):
        self.stop = False
        try:
            import threading

            import pynvml as N

            N.nvmlInit()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
            try:
                self.p = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                     "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except FileNotFoundError:
                self.p = None
        return self

    def __exit__(self, *exc):
        if self.thread is not None:
            self.stop = True
            self.thread.join(timeout=5)
        if self.p is not None:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()
                out, _ = self.p.communicate()
            names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
            for ln in out.splitlines():
                f = [x.strip() for x in ln.split(",")]
                if len(f) < 8:
                    continue
                try:
                    self.sm.append(float(f[0]))
                    self.mx = float(f[1])
                except ValueError:
                    continue
                self.reasons.update(n for n, v in zip(names, f[4:8]) if v.lower().startswith("active"))

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml, 1 ms polling" if self.thread is not None else "nvidia-smi"}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def run_ours(args, ws, rank, local):
    import torch

    from paper_2601_11546_b200 import _abi, _marshal
    from paper_2601_11546_b200._native import NativeEngine
    from paper_2601_11546_b200.engine import Engine

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    pool = args.config == "5"  # one trace sharded over the ranks (or over CTAs on one GPU)
    trace, world, cfg, wname = workload(args.config, seed=0 if pool else rank)
    I = args.iters_per_step
    stream = torch.cuda.current_stream(dev)
    if pool:
        shards, srank = (ws, rank) if ws > 1 else (args.shards or 8, -1)
    else:
        shards, srank = 1, -1

    # ---- device-resident timing (inputs already in HBM)
    m = _marshal.marshal_trace(trace, cfg.block_size, "relserve", world, None)
    ne = NativeEngine([m.view], _marshal.make_config(cfg, "relserve"), _marshal.make_model(world),
                      _marshal.make_model(world), [_marshal.dpu_rng_state(0)], local,
                      log_capacity=I * (args.steps + args.warmup + 1) + WINDOW_START, shards=shards, rank=srank)
    if pool and ws > 1:
        from paper_2601_11546_b200 import sharded

        ne.connect(sharded.exchange_handles(ne.mailbox_handle()))
    ne.step(WINDOW_START, stream)
    st = ne.status(stream)[0]
    assert st.status == _abi.RS_RUNNING and st.iterations == WINDOW_START, (st.status, st.iterations)
    n_read = st.n_log
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        ne.step(I, stream)
    st = ne.status(stream)[0]
    n_read = st.n_log
    it0 = st.iterations
    ph0 = list(st.phase_cycles)
    ab0 = st.alg_bytes
    pending0 = trace.columns().num_requests
    evs = []
    recs = []
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ne.step(I, stream)
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    st = ne.status(stream)[0]
    iters = st.iterations - it0
    ph = [a - b for a, b in zip(st.phase_cycles, ph0)]
    alg_window = st.alg_bytes - ab0
    assert st.status == _abi.RS_RUNNING, f"trace ended inside the window (status {st.status})"
    recs = ne.read_log(0, n_read, st.n_log - n_read)
    recs_all = ne.read_log(0, 0, st.n_log)
    gen, pre, comp, prio = ne.read_requests(0, trace.columns().num_requests)
    pending_end = int((pre == 0).sum())
    ne.close()
    it1 = it0 + iters
    wstats = window_stats(recs_all, comp, trace.columns(), it0, it1)
    t_ms = sum(step_ms)
    t_max = max_over_ranks(t_ms, ws, dev)
    # independent traces: every rank's iterations count; one sharded pool: its iterations once
    total_iters = float(iters) if pool else sum_over_ranks(float(iters), ws, dev)
    value = total_iters / (t_max / 1e3)
    c = trace.columns()
    per_launch_bytes = alg_window / args.steps
    avg_launch_s = (t_ms / args.steps) / 1e3
    peak, peak_kind = peaks()
    achieved = per_launch_bytes / avg_launch_s / 1e9
    achieved_b_iter = b_iter(wstats) * (iters / args.steps) / avg_launch_s / 1e9
    traffic_launch, traffic_src = traffic(args.config, I)

    # ---- end to end through the public API (host buffers, copies inside)
    e2e = None
    if not args.no_e2e:
        e2e = e2e_runs(args, trace, world, cfg, m, dev, local, stream, ws, pool, shards, srank, it1)

    out = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and ws == 1:
            cpu = cpu_baseline(args, trace, world, cfg)
        out = {
            "metric": METRIC,
            "value": value,
            "unit": "iters/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": t_max / args.steps,
            "higher_is_better": True,
            "scaling": "strong" if pool else "weak",
            "vs_baseline": None,
            "dtype": "f64+int32",
            "data": "synthetic (relsim generate_trace, count-identical to the reference generator)",
            "config": config_dict(wname, I, it0, it1, wstats),
            "run": {"shards": shards, "shard_mode": ("one per GPU (NVLink P2P mailboxes)" if pool and ws > 1
                                                      else "CTAs of one launch on one GPU" if pool else None),
                    "requests_total": pending0, "pending_requests_end": pending_end,
                    "live_requests_mean": wstats["live_requests_mean"],
                    "live_relqueries_mean": wstats["live_relqueries_mean"],
                    "traces_per_gpu": 1 if not pool else None},
            "iterations_timed": int(total_iters),
            "e2e": e2e,
            "gpu_launches": args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic_launch, "peak_source": peak_kind,
                         "alg_bytes_per_iter": alg_window / max(1, iters),
                         "b_iter": b_iter(wstats), "achieved_b_iter": achieved_b_iter,
                         "frac_b_iter": achieved_b_iter / peak,
                         "traffic_source": traffic_src,
                         "note": "latency-bound: one dependent iteration chain per trace. frac: the bytes this "
                                 "design moves, counted on the device (DESIGN.md 5); frac_b_iter: SURVEY 8d's "
                                 "declared B_iter = 6 N_live + 56 R_live (a design rescanning every live row each "
                                 "iteration) at the same iteration rate; traffic: ncu dram bytes per launch "
                                 "(profiles/traffic.json)"},
            "clocks": clk.summary(),
            "phase_cycles_per_iter": dict(zip(PHASES, [round(x / max(1, iters), 1) for x in ph])),
            "iteration_mix": {"prefill": int((recs["action"] == 0).sum()), "decode": int((recs["action"] == 1).sum()),
                              "idle": int((recs["action"] == 2).sum()),
                              "reestimated_per_iter": float(recs["n_reestimated"].mean()) if len(recs) else 0.0},
            "cpu_baseline": cpu,
        }
    return out


#: end-to-end repetitions: the host-side parts (engine creation, result collection) see OS
#: noise of several ms, so the run is repeated and the median reported (every run listed)
E2E_REPEATS = 3


def e2e_runs(args, trace, world, cfg, m, dev, local, stream, ws, pool, shards, srank, it_end):
    """The bench window through the public `Engine` API from host arrays: trace upload and
    first-sight kernel (engine creation), every step's launch + status + decision-record
    readback, and the final ledger / completion readback, wall-clock timed."""
    import gc

    import torch

    from paper_2601_11546_b200.engine import Engine

    I = args.iters_per_step
    trace.pin_memory()  # the caller's host buffers are page-locked (outside the timed region)
    c = trace.columns()
    runs = []
    for rep in range(E2E_REPEATS + 1):  # run 0: untimed warm-up of the host path (allocator, first-call costs)
        torch.cuda.synchronize(dev)
        gc.collect()
        t0 = time.perf_counter()
        eng = Engine(trace, "relserve", world, cfg, seed=0, device=local, stream=stream, shards=shards,
                     shard_rank=srank)
        if pool and ws > 1:
            from paper_2601_11546_b200 import sharded

            sharded.connect(eng)
        t1 = time.perf_counter()
        eng.step(WINDOW_START)
        t15 = time.perf_counter()
        eng.step(it_end - eng.iteration)  # up to the device window's last iteration (the API launches in chunks)
        t2 = time.perf_counter()
        eng._collect(0.0)
        torch.cuda.synchronize(dev)
        t3 = time.perf_counter()
        e_iters = eng.iteration
        eng.close()
        wall = max_over_ranks(t3 - t0, ws, dev)
        total = float(e_iters) if pool else sum_over_ranks(float(e_iters), ws, dev)
        if rep == 0:
            continue
        runs.append({"value": total / wall, "wall_s": wall, "iterations": int(e_iters),
                     "breakdown_ms": {"create_ms": 1e3 * (t1 - t0), "admission_steps_ms": 1e3 * (t15 - t1),
                                      "steps_ms": 1e3 * (t2 - t15),
                                      "collect_ms": 1e3 * (t3 - t2)}})
    med = sorted(runs, key=lambda r: r["value"])[len(runs) // 2]
    h2d = sum(v.nbytes for v in m.arrays.values() if v is not None)
    # bytes per bench step (I iterations) of the run: the trace upload and the final readback
    # spread over the run's iterations, plus each iteration's 96-byte decision record
    n_launch = -(-(it_end - WINDOW_START) // Engine.chunk_iterations) + 1
    d2h_total = it_end * 96 + n_launch * 128 + c.num_requests * 4 + c.num_relqueries * 32
    return {"value": med["value"], "unit": "iters/s",
            "h2d_bytes_per_step": int(h2d * I / it_end), "d2h_bytes_per_step": int(d2h_total * I / it_end),
            "window": [0, it_end],
            "iterations": med["iterations"], "wall_s": med["wall_s"], "breakdown_ms": med["breakdown_ms"],
            "runs": [{"value": round(r["value"], 1), **{k: round(v, 2) for k, v in r["breakdown_ms"].items()}}
                     for r in runs],
            "statistic": f"median of {E2E_REPEATS} runs after one untimed warm-up run",
            "includes": "trace upload, iterations 0..the device window's end (incl. first-sight DPU), per-step "
                        "record readback, final ledger/completion readback"}


def cpu_baseline(args, trace, world, cfg, iters=None):
    """Oracle (C restatement of the reference loop, 1 thread) on the same trace."""
    from dataclasses import replace

    from oracle import oracle

    iters = iters or (args.cpu_iters if args.config in ("2", "3") else min(args.cpu_iters, 1000))
    c2 = replace(cfg, iteration_limit=WINDOW_START + iters)
    t0 = time.perf_counter()
    r = oracle.run(trace, "relserve", world, c2, None, 0)
    wall = time.perf_counter() - t0
    win = r.iter_wall[WINDOW_START:WINDOW_START + iters]
    return {"value": float(len(win) / win.sum()), "unit": "iters/s", "cores": 1, "kind": "port",
            "sample": f"iterations [{WINDOW_START}, {WINDOW_START + len(win)}) of the same trace "
                      f"(steady state; first-sight iteration {r.first_sight_iter} took "
                      f"{r.first_sight_wall_s:.3f} s); run wall {wall:.1f} s",
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, ws, rank):
    if rank != 0:
        return None
    trace, world, cfg, wname = workload(args.config, seed=0)
    per_step = max(1, args.iters_per_step)
    n = WINDOW_START + (args.warmup + args.steps) * per_step
    from dataclasses import replace

    from oracle import oracle

    r = oracle.run(trace, "relserve", world, replace(cfg, iteration_limit=n), None, 0)
    lo = WINDOW_START + args.warmup * per_step
    win = r.iter_wall[lo:n]
    value = float(len(win) / win.sum())
    wstats = window_stats(r.log, r.completion_iter, trace.columns(), lo, n)
    return {
        "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": float(win.sum() / args.steps * 1e3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+int32",
        "data": "synthetic (relsim generate_trace, count-identical to the reference generator)",
        "config": config_dict(wname, per_step, lo, n, wstats),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": 1, "kind": "port",
                         "sample": f"oracle/ C restatement of relsim Engine.run, iterations [{lo}, {n})",
                         "cpu": _cpu_model()},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def config4_cells():
    """2 cost models x 16 rates (0.25..4.0) x 32 size ranges (1, s),
    s geometric 8..1000; 100 relQueries each; seed = cell index."""
    rates = np.geomspace(0.25, 4.0, 16)
    sizes = np.unique(np.round(np.geomspace(8, 1000, 32)).astype(int))
    while len(sizes) < 32:  # keep 32 distinct ranges
        sizes = np.unique(np.append(sizes, sizes[-1] + len(sizes)))
    cells = []
    for model in ("opt-13b-like", "llama-70b-like"):
        for r in rates:
            for s in sizes[:32]:
                cells.append((model, float(r), int(s)))
    return cells


def run_config4(args, ws, rank, local):
    """Independent full runs of config-4 cells: one CTA per trace, 128 traces per GPU."""
    import torch

    from paper_2601_11546_b200 import EngineConfig, TraceConfig, _abi, _marshal, generate_trace, world_preset
    from paper_2601_11546_b200._native import NativeEngine

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cells = config4_cells()
    # an 8-way partition of the 1,024 cells (interleaved, so every share mixes models, rates, sizes)
    mine = list(range(rank, len(cells), 8))[: args.traces_per_gpu]
    cfg = EngineConfig()
    by_model = {}
    for ci in mine:
        model, rate, s = cells[ci]
        t = generate_trace(TraceConfig(num_relqueries=100, size_range=(1, s), rate=rate, seed=ci)).pin_memory()
        by_model.setdefault(model, []).append((ci, t))
    # engines of GROUP traces of one cost model, the most decode work (sum of output tokens, the
    # best predictor of a trace's iteration count) first: in the end-to-end pass an engine is
    # launched as soon as it is built, so the long traces start first and later engines are built
    # while earlier ones run
    GROUP = 8
    work = lambda it: -int(it[1].columns().out.sum())  # noqa: E731
    groups = []
    for model, items in by_model.items():
        items.sort(key=work)
        groups += [(model, items[k:k + GROUP]) for k in range(0, len(items), GROUP)]
    groups.sort(key=lambda g: work(g[1][0]))
    if len(groups[0][1]) > 1:  # the longest trace alone in the first engine: it is built and started soonest
        m0, g0 = groups[0]
        groups = [(m0, g0[:1]), (m0, g0[1:])] + groups[1:]
    worlds = {m: world_preset(m) for m in by_model}
    c_cfg = _marshal.make_config(cfg, "relserve")

    def make_engine(model, items):
        w = worlds[model]
        ms = [_marshal.marshal_trace(t, cfg.block_size, "relserve", w) for _, t in items]
        ne = NativeEngine([m.view for m in ms], c_cfg, _marshal.make_model(w), _marshal.make_model(w),
                          [_marshal.dpu_rng_state(ci) for ci, _ in items], local, log_capacity=0)
        return ne, ms

    streams = [torch.cuda.Stream(dev) for _ in groups]
    main_s = torch.cuda.current_stream(dev)

    def collect(engines, order=None):
        iters, alg, d2h = 0, 0, 0
        pairs = list(zip(engines, streams))
        for (ne, ms), st in (pairs if order is None else [pairs[k] for k in order]):
            for s_ in ne.status(st):
                assert s_.status == _abi.RS_OK, s_.status
                iters += s_.iterations
                alg += s_.alg_bytes
            R = sum(m.view.num_relqueries for m in ms)
            N = sum(m.view.num_requests for m in ms)
            out = ne.read_results(R, N, st)
            d2h += sum(x.nbytes for x in out)
        return iters, alg, d2h

    def device_sweep():
        """Every trace of this GPU's share run to completion from engines built beforehand (inputs
        resident): the events bracket the launches only."""
        engines = [make_engine(m, it) for m, it in groups]
        torch.cuda.synchronize(dev)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(main_s)
        for (ne, _), st in zip(engines, streams):
            st.wait_event(a)
            ne.step(1 << 30, st)  # one launch runs every trace of the engine to completion
            e = torch.cuda.Event()
            e.record(st)
            main_s.wait_event(e)
        b.record(main_s)
        torch.cuda.synchronize(dev)
        iters, alg, _ = collect(engines)
        for ne, _ in engines:
            ne.close()
        return a.elapsed_time(b) / 1e3, iters, alg

    def e2e_sweep():
        """The public API end to end, wall clock: per engine, the host trace columns are marshalled,
        uploaded (engine creation, first-sight kernels) and launched at once; then every engine's
        status and results (ledgers + completion iterations) come back."""
        t0 = time.perf_counter()
        engines = []
        for (m, it), st in zip(groups, streams):
            ne, ms = make_engine(m, it)
            ne.step(1 << 30, st)
            engines.append((ne, ms))
        t1 = time.perf_counter()
        # the engines with the least work finish first: read them while the longest still run
        iters, _, d2h = collect(engines, order=range(len(engines) - 1, -1, -1))
        t2 = time.perf_counter()
        h2d = sum(v.nbytes for _, ms in engines for m_ in ms for v in m_.arrays.values() if v is not None)
        for ne, _ in engines:
            ne.close()
        return t2 - t0, t1 - t0, iters, h2d, d2h

    for _ in range(args.warmup):
        device_sweep()
        e2e_sweep()
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()
    dev_s, iters, alg, e2e_s, create_s, d2h, h2d, e_iters = 0.0, 0, 0, 0.0, 0.0, 0, 0, 0
    t0 = time.perf_counter()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            d, n, ab = device_sweep()
            dev_s += d
            iters += n
            alg += ab
            w, cr, en, ib, ob = e2e_sweep()
            e2e_s += w
            create_s += cr
            e_iters += en
            h2d += ib
            d2h += ob
    wall = time.perf_counter() - t0
    t_max = max_over_ranks(dev_s, ws, dev)
    e2e_max = max_over_ranks(e2e_s, ws, dev)
    total = sum_over_ranks(float(iters), ws, dev)
    e_total = sum_over_ranks(float(e_iters), ws, dev)
    alg_total = sum_over_ranks(float(alg), ws, dev)
    if rank != 0:
        return None
    peak, peak_kind = peaks()
    achieved = alg_total / t_max / 1e9 / ws  # per GPU
    e2e = {"value": e_total / e2e_max, "unit": "iters/s", "h2d_bytes_per_step": int(h2d / args.steps),
           "d2h_bytes_per_step": int(d2h / args.steps),
           "breakdown_ms": {"build_and_launch_ms_per_step": 1e3 * create_s / args.steps,
                            "total_ms_per_step": 1e3 * e2e_s / args.steps},
           "includes": "per step: marshal of the host trace columns, upload + first-sight kernels (engine "
                       "creation) and launch of each engine (largest traces first; later engines are built while "
                       "earlier ones run), then every engine's status and its ledger + completion readback"}
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        cpu = cpu_baseline_config4([cells[ci] + (ci,) for ci in mine])
    return {
        "metric": "sched iters/sec, config-4 sweep (aggregate over independent traces)",
        "value": total / t_max, "unit": "iters/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64+int32", "data": "synthetic (generate_trace per config-4 cell)",
        "config": {"workload": f"config4: {args.traces_per_gpu} traces/GPU of 100 relQ, sizes (1,s) s=8..1000, "
                               "rates 0.25..4, opt-13b/llama-70b, full runs; a step = every trace of the share "
                               "run to completion", "traces_per_gpu": len(mine), "engines": len(groups),
                   "l2": "working set of each step is fresh (engines rebuilt between steps)"},
        "iterations_timed": int(total), "gpu_launches": len(groups) * args.steps, "clocks": clk.summary(),
        "host_wall_s": wall, "cpu_baseline": cpu, "e2e": e2e,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "peak_source": peak_kind,
                     "note": "device-counted algorithmic bytes of all traces / the step's device time; "
                             "latency-bound (one dependent iteration chain per trace, 128 CTAs on 148 SMs)"},
    }


def _cpu_cell(cell):
    """One config-4 cell on the oracle (child process of cpu_baseline_config4)."""
    import time as _t

    from oracle import oracle
    from paper_2601_11546_b200 import EngineConfig, TraceConfig, generate_trace, world_preset

    model, rate, s, ci = cell
    t = generate_trace(TraceConfig(num_relqueries=100, size_range=(1, s), rate=rate, seed=ci))
    t0 = _t.perf_counter()
    r = oracle.run(t, "relserve", world_preset(model), EngineConfig(), None, ci)
    return r.iterations, _t.perf_counter() - t0


def cpu_baseline_config4(cells):
    """the oracle over the same cells, full runs, a process pool over all host cores
    (the reference's `relsim run --jobs` pattern, cli.py:194-196)."""
    import multiprocessing as mp

    n = os.cpu_count() or 1
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(n) as pool:
        res = pool.map(_cpu_cell, cells, chunksize=1)
    wall = time.perf_counter() - t0
    iters = sum(r[0] for r in res)
    return {"value": iters / wall, "unit": "iters/s", "cores": n, "kind": "port",
            "sample": f"the same {len(cells)} cells, full runs, {n}-process pool; {iters} iterations in {wall:.1f} s "
                      "(incl. pool start-up)", "cpu": _cpu_model()}


def main():
    args = parse()
    ws, rank, local = dist_init(args)
    if args.impl == "reference":
        out = run_reference(args, ws, rank)
    elif args.config == "4":
        out = run_config4(args, ws, rank, local)
    else:
        out = run_ours(args, ws, rank, local)
    if rank == 0 and out is not None:
        print(json.dumps(out))
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
