#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/full
O=gpurun_out/full
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > $O/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python bench.py > $O/bench_c2.json 2> $O/bench.err
python bench.py --impl reference > $O/bench_ref_c2.json 2>> $O/bench.err
python bench.py --config 3 > $O/bench_c3.json 2>> $O/bench.err
python bench.py --config 3 --impl reference > $O/bench_ref_c3.json 2>> $O/bench.err
python bench.py --config 5 --shards 8 > $O/bench_c5_s8.json 2>> $O/bench.err
python bench.py --config 5 --shards 1 --no-cpu-baseline > $O/bench_c5_s1.json 2>> $O/bench.err
python bench.py --config 4 > $O/bench_c4.json 2>> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --no-cpu-baseline --no-e2e > $O/ncu_launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:engine_kernel -s 2 -c 1 -o $O/prof_c2 python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 1 > $O/ncu_full_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:first_sight -c 1 -o $O/prof_fs_c5 python bench.py --config 5 --shards 1 --no-cpu-baseline --no-e2e --steps 2 --warmup 1 > $O/ncu_fs_run.log 2>&1
