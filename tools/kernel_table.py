"""Per-kernel HBM roofline table: every kernel of this repository, timed and DRAM-counted by ncu.

    # on the GPU box: the workloads, under ncu's per-launch metrics (cold-cache, serialised)
    for w in c2 c5 c3p; do
      ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
          --clock-control none --csv --log-file gpurun_out/kernels_$w.csv python tools/kernel_table.py run $w
    done
    # here: the table
    python tools/kernel_table.py table profiles/r2/kernels.md profiles/r2/kernels/kernels_{c2,c5,c3p}.csv

`run` drives each kernel family once on its natural workload:
  * config 2 (10^6 requests): engine creation (row checks, static order, first sight) + 2 launches of
    250 scheduler iterations (engine_kernel, the common-configuration instantiation);
  * config 5 (8*10^6 requests, 8 shards as CTAs of one launch): creation + 1 launch of 100 iterations;
  * config 3 in parity mode (5,000 relQueries): 20 iterations recording the full waiting order, which
    the device radix sort rebuilds each iteration (the general engine_kernel instantiation).
`table` aggregates the ncu CSV per kernel: launches, mean duration, mean DRAM bytes, achieved DRAM GB/s,
and that as a fraction of MEASURED_PEAKS.json's copy bandwidth (the burst figure: each launch is timed
alone by ncu).  The scheduler kernel is latency-bound (one dependent iteration chain per trace),
so its fraction is small by construction; the creation kernels are the bandwidth-shaped ones.
"""

import csv
import io
import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def run(w: str):
    import torch

    import bench
    from paper_2601_11546_b200 import _marshal
    from paper_2601_11546_b200._native import NativeEngine
    from paper_2601_11546_b200.engine import Engine
    from paper_2601_11546_b200 import SimulationAborted

    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    for cfg_id, shards, iters, launches in {"c2": [("2", 1, 250, 2)], "c5": [("5", 8, 100, 1)], "c3p": []}[w]:
        trace, world, cfg, _ = bench.workload(cfg_id, seed=0)
        m = _marshal.marshal_trace(trace, cfg.block_size, "relserve", world, None)
        ne = NativeEngine([m.view], _marshal.make_config(cfg, "relserve"), _marshal.make_model(world),
                          _marshal.make_model(world), [_marshal.dpu_rng_state(0)], 0,
                          log_capacity=iters * launches + 8, shards=shards, rank=-1)
        for _ in range(launches):
            ne.step(iters, stream)
        ne.status(stream)
        torch.cuda.synchronize()
        ne.close()
        print(f"config {cfg_id}: {launches} x {iters} iterations", flush=True)
    if w != "c3p":
        return
    trace, world, cfg, _ = bench.workload("3", seed=0)
    cfg.iteration_limit = 20
    e = Engine(trace, "relserve", world, cfg, None, 0, device=0, record_waiting_order=True)
    try:
        e.run()
    except SimulationAborted:  # the iteration limit
        pass
    e.close()
    print("config 3 parity mode: 20 iterations", flush=True)


WORKLOAD = {"c2": "config 2", "c5": "config 5, 8 shards", "c3p": "config 3, parity mode"}


def table(out_md: str, *csv_paths: str):
    per = defaultdict(lambda: defaultdict(float))
    seen = defaultdict(set)
    for csv_path in csv_paths:
        w = Path(csv_path).stem.split("_")[-1]
        text = Path(csv_path).read_text()
        text = text[text.index('"ID"'):] if '"ID"' in text else text
        for r in csv.DictReader(io.StringIO(text)):
            if r["Kernel Name"].startswith("void at::"):  # torch's own fills
                continue
            name = (WORKLOAD.get(w, w), r["Kernel Name"])
            v = float(r["Metric Value"].replace(",", "")) * UNITS.get(r["Metric Unit"], 1)
            per[name][r["Metric Name"]] += v
            seen[name].add(r["ID"])
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (
        ROOT / "MEASURED_PEAKS.json").exists() else 6553.9
    lines = ["| workload | kernel | launches | mean duration (µs) | DRAM bytes / launch | L2 bytes / launch | DRAM GB/s | "
             "frac of %.0f GB/s |" % peak, "|---|---|---|---|---|---|---|---|"]
    summary = []
    for (w, name), d in sorted(per.items(), key=lambda kv: (kv[0][0], -kv[1]["gpu__time_duration.sum"])):
        n = len(seen[(w, name)])
        if not d["gpu__time_duration.sum"]:
            continue
        t = d["gpu__time_duration.sum"] / n
        dram = (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / n
        l2 = d["lts__t_bytes.sum"] / n
        gbs = dram / t / 1e9 if t else 0.0
        short = name.split("(")[0].replace("void ", "")
        lines.append(f"| {w} | `{short}` | {n} | {t * 1e6:.1f} | {dram:,.0f} | {l2:,.0f} | {gbs:.0f} | {gbs / peak:.3f} |")
        summary.append(dict(workload=w, kernel=short, launches=n, us=t * 1e6, dram_bytes=dram, l2_bytes=l2, gbs=gbs,
                            frac=gbs / peak))
    head = ["# Every kernel of the repository: ncu duration and DRAM traffic per launch", "",
            "Generated by `tools/kernel_table.py` (its docstring has the commands) from ncu's per-launch metrics "
            "(`gpu__time_duration.sum`, `dram__bytes_read.sum + dram__bytes_write.sum`, `lts__t_bytes.sum`; "
            "cold-cache, serialised launches, `--clock-control none`); raw CSVs in `kernels/`.  DRAM GB/s = DRAM "
            "bytes / duration, against MEASURED_PEAKS.json's copy bandwidth.  `engine_kernel` is one persistent "
            "CTA running hundreds of dependent scheduler iterations per launch (latency-bound, DESIGN.md 5: "
            "its yardstick is cycles per iteration); the creation kernels (`validate_rows_kernel`, "
            "`first_sight_seg_kernel`, `first_sight_sum_kernel`) stream the trace columns once; the radix-sort "
            "kernels order the static waiting queue at creation and, in parity mode, every recorded iteration's "
            "full waiting queue.", ""]
    Path(out_md).write_text("\n".join(head + lines) + "\n")
    Path(out_md).with_suffix(".json").write_text(json.dumps(dict(peak_gbs=peak, kernels=summary), indent=1))
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        table(*sys.argv[2:])
