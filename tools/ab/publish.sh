#!/bin/bash
# copy gpurun_out/full into profiles/r1 (+ ncu summaries)
cd "$(dirname "$0")/../.."
O=gpurun_out/full; P=profiles/r1
cp $O/bench_c2.json $P/bench_config2.json; cp $O/bench_c3.json $P/bench_config3.json; cp $O/bench_c4.json $P/bench_config4.json
cp $O/bench_c5_s8.json $P/bench_config5_8shards.json; cp $O/bench_c5_s1.json $P/bench_config5_unsharded.json
cp $O/bench_ref_c2.json $P/bench_reference_config2.json; cp $O/bench_ref_c3.json $P/bench_reference_config3.json
cp $O/pytest_gpu.log $P/pytest_gpu.log; cp $O/smoke.log $P/smoke.log; cp $O/launches_c2.csv profiles/r1_launches_engine_config2.csv
ncu -i $O/prof_c2.ncu-rep --page raw --csv > /tmp/raw.csv 2>/dev/null
python - <<'PY'
import csv
rows=list(csv.reader(open('/tmp/raw.csv')))
hdr, units, vals = rows[0], rows[1], rows[2]
want=["dram__bytes_read.sum","dram__bytes_write.sum","gpu__time_duration.sum","l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct","launch__registers_per_thread","launch__shared_mem_per_block_dynamic","lts__t_sectors.sum","lts__t_bytes.sum","sm__icc_requests.sum","sm__icc_request_hit_rate.pct","sm__warps_active.avg.pct_of_peak_sustained_active","smsp__inst_executed.sum","sm__cycles_elapsed.avg","launch__grid_size","launch__block_size","smsp__pcsamp_sample_count"]
out=[f"{h} {units[i]} {vals[i]}" for w in want for i,h in enumerate(hdr) if h==w]
open('profiles/r1/engine_kernel_raw.txt','w').write("\n".join(out)+"\n")
print("\n".join(out))
PY
ncu -i $O/prof_c2.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_full.csv 2>/dev/null
python tools/ncu_lines.py /tmp/src_full.csv 250 40 > $P/engine_kernel_lines.txt 2>/dev/null
python tools/ncu_hot_lines.py /tmp/src_full.csv 250 30 > $P/engine_kernel_hot_lines.txt 2>/dev/null
head -2 $P/engine_kernel_lines.txt; head -2 $P/engine_kernel_hot_lines.txt
python - <<'PY'
import csv
rows=list(csv.reader(open('/tmp/src_full.csv')))
idx=None; tot={}
for r in rows:
    if r and r[0]=="Line No": idx={h:i for i,h in enumerate(r)}; continue
    if r and r[0]=="Address": break
    if idx and r and r[0] not in("","Function Name"):
        for h,i in idx.items():
            if h.startswith('stall_') and 'Not Issued' not in h:
                try: tot[h]=tot.get(h,0)+int(r[i])
                except: pass
print(sorted(tot.items(), key=lambda x:-x[1])[:8])
PY
grep -E "engine_kernel" $O/launches_c2.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '; echo
grep -E "first_sight" $O/launches_c2.csv | awk -F'","' '{print $NF}' | tr -d '"'
