cd /root/repo
for v in base ph2; do for s in 1 8; do
RS_LIB=scratch/lib_$v.so timeout 300 python bench.py --config 5 --shards $s --no-cpu-baseline --no-e2e > gpurun_out/c5_${v}_s$s.json 2>&1
done; done
