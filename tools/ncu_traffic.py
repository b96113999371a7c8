"""Summarise an `ncu --set full` capture of one kernel launch for profiles/.

    python tools/ncu_traffic.py REPORT.ncu-rep CONFIG ITERS_PER_LAUNCH OUT_SUMMARY.json

Writes the launch's duration, DRAM and L2 bytes, occupancy, local-memory
traffic and the warp-stall sample breakdown to OUT_SUMMARY.json, and records
the DRAM bytes per launch under "config<CONFIG>" in profiles/traffic.json
(bench.py's roofline.traffic).  ITERS_PER_LAUNCH: scheduler iterations the
captured launch ran (engine_kernel), or 0 for a creation kernel.
"""

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1, "second": 1, "nsecond": 1e-9}


def raw(report: str) -> dict:
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    d = {}
    for k, u, v in zip(head, units, rows[2]):
        try:
            d[k] = float(v.replace(",", "")) * UNITS.get(u, 1)
        except ValueError:
            d[k] = v
    return d


def main():
    report, cfg, iters, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), Path(sys.argv[4]).resolve()
    d = raw(report)
    dram = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    stalls = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: int(v) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued") and v}
    n = sum(stalls.values()) or 1
    summ = {
        "report": Path(report).name,
        "kernel": d["Kernel Name"],
        "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size"),
        "registers_per_thread": d.get("launch__registers_per_thread"),
        "duration_s": d["gpu__time_duration.sum"],
        "iters_per_launch": iters,
        "us_per_iteration": d["gpu__time_duration.sum"] / iters * 1e6 if iters else None,
        "dram_bytes_per_launch": dram,
        "l2_bytes_per_launch": d["lts__t_sectors.sum"] * 32,
        "dram_bytes_per_iteration": dram / iters if iters else None,
        "l2_bytes_per_iteration": d["lts__t_sectors.sum"] * 32 / iters if iters else None,
        "dram_throughput_GBps": dram / d["gpu__time_duration.sum"] / 1e9,
        "warps_active_pct": d.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "local_load_sectors": d.get("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum"),
        "local_store_sectors": d.get("l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum"),
        "inst_executed": d.get("smsp__inst_executed.sum"),
        "stall_samples": n,
        "stall_share": {k: round(v / n, 4) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])},
    }
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_text(json.dumps(summ, indent=1) + "\n")
    tf = ROOT / "profiles" / "traffic.json"
    t = json.loads(tf.read_text()) if tf.exists() else {}
    key = f"config{cfg}" if iters else f"config{cfg}_creation"
    t[key] = {"kernel": summ["kernel"], "dram_bytes_per_launch": dram, "l2_bytes_per_launch":
              summ["l2_bytes_per_launch"], "iters_per_launch": max(iters, 1), "capture": str(out.relative_to(ROOT))}
    tf.write_text(json.dumps(t, indent=1) + "\n")
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
