#!/bin/bash
# the fused selection's DRAM / L2 traffic in the step's real cache state
# (application replay, no cache control: every pass runs after an attention)
mkdir -p gpurun_out
timeout -k 10 600 ncu --replay-mode application --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__t_sectors_srcunit_tex.sum -k regex:"k_select_fused|k_attend" --launch-skip 30 -c 4 --csv --log-file gpurun_out/selncu.csv python bench.py --steps 6 --warmup 4 --e2e-steps 1 --no-cpu --no-extra --max-iters 2 > gpurun_out/selncu.log 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/selncu.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
for r in rows[1:]: print(r[ki][:28], r[mi], r[vi])
PY
tail -3 gpurun_out/selncu.log
