#!/bin/bash
# alternate variants R rounds: scratch/abx.sh R name1 name2 ... -> gpurun_out/abx_<name>_c<cfg>_<round>.json
cd "$(dirname "$0")/../.."
R=$1; shift
for r in $(seq 1 $R); do
  for n in "$@"; do
    for cfg in ${CFGS:-2 3}; do
      RS_LIB=scratch/lib_$n.so timeout 300 python bench.py --config $cfg --shards 1 --no-cpu-baseline --no-e2e > gpurun_out/abx_${n}_c${cfg}_$r.json 2>&1
    done
  done
done
