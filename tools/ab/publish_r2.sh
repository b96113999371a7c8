#!/bin/bash
# copy gpurun_out/full (tools/ab/full_measurement.sh) into profiles/r2 and refresh the ncu summaries
# (profiles/traffic.json feeds bench.py's roofline.traffic)
cd "$(dirname "$0")/../.."
O=gpurun_out/full; P=profiles/r2
for f in bench_c2 bench_c3 bench_c4 bench_c5_s1 bench_c5_s8 bench_ref_c2 bench_ref_c3; do
  tail -1 $O/$f.json > $P/$f.json
done
cp $O/pytest_gpu.log $P/pytest_gpu.log; cp $O/smoke.log $P/smoke.log; cp $O/launches_c2.csv $P/launches_engine_config2.csv
python tools/ncu_traffic.py $O/prof_c2.ncu-rep 2 250 $P/engine_kernel_config2.json > /dev/null
python tools/ncu_traffic.py $O/prof_fs_c5.ncu-rep 5 0 $P/first_sight_config5.json > /dev/null
python - <<'PY'
import json
for f in ["engine_kernel_config2", "first_sight_config5"]:
    d = json.load(open(f"profiles/r2/{f}.json"))
    print(f, d["kernel"][:40], "us/launch %.1f" % (d["duration_s"] * 1e6), "us/iter", d["us_per_iteration"],
          "dram/launch", d["dram_bytes_per_launch"], "l2/launch", d["l2_bytes_per_launch"], list(d["stall_share"].items())[:4])
PY
