#!/bin/bash
# alternate library variants through bench.py's e2e leg: tools/ab/e2e_ab.sh R name1 name2 ...
cd "$(dirname "$0")/../.."
R=$1; shift
for r in $(seq 1 $R); do
  for n in "$@"; do
    RS_LIB=scratch/lib_$n.so timeout 300 python bench.py --no-cpu-baseline > gpurun_out/e2e_${n}_$r.json 2>&1
  done
done
