cd /root/repo
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_sweep.py tests/test_gpu_fullscale.py tests/test_gpu_units.py -q -x -m gpu > gpurun_out/t_fs.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:first_sight python bench.py --config 5 --shards 1 --no-cpu-baseline --no-e2e --steps 2 --warmup 1 > gpurun_out/ncu_fs.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:first_sight_seg -c 1 -o gpurun_out/prof_fs2_c5 python bench.py --config 5 --shards 1 --no-cpu-baseline --no-e2e --steps 2 --warmup 1 > /dev/null 2>&1
