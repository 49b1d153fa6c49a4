#!/bin/bash
# select / attend durations with warm caches (ncu --cache-control none: the
# persisting-L2 centroids stay resident as in the stream), and the unfused
# selection's per-warp phase times
mkdir -p gpurun_out
timeout -k 10 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum --cache-control none --clock-control none -k regex:"k_select|k_attend" --launch-skip 40 -c 6 --csv --log-file gpurun_out/selwarm.csv python bench.py --steps 10 --warmup 5 --e2e-steps 2 --no-cpu --no-extra --max-iters 4 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/selwarm.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
for r in rows[1:]: print(r[ki][:40], r[mi], r[vi])
PY
export CKV_LIB=$PWD/paper_2412_03213_b200/libckv_b200_seldbg.so
CKV_SELECT_UNFUSED=1 CKV_DEBUG_TIMING=1 timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu --no-extra --max-iters 4 2>&1 | grep "k_select dbg" | tail -3
