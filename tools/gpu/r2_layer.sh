#!/bin/bash
timeout 600 python tools/layer_prof.py 20 8
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_select|k_attend|k_append|k_score" --launch-skip 300 -c 80 --csv --log-file gpurun_out/layer_launch.csv python tools/layer_prof.py 4 8 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/layer_launch.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size') if 'Grid Size' in h else None
agg=collections.defaultdict(list)
for r in rows[1:]:
    agg[(r[ki][:60], r[gi] if gi else '')].append(float(r[vi].replace(',','')))
for k,v in agg.items(): print(f"{k[0]:60s} grid={k[1]:14s} n={len(v):3d} mean={sum(v)/len(v)/1000:.2f} us")
PY
