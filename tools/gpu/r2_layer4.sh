#!/bin/bash
mkdir -p gpurun_out
unset CKV_SEL_FEW
for n in 2 4 8; do echo "NC=$n: $(CKV_SEL_NC=$n timeout -k 10 300 python tools/layer_prof.py 20 8 2>&1 | tail -1)"; done
timeout -k 10 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_select|k_attend|k_append|k_score" --launch-skip 300 -c 60 --csv --log-file gpurun_out/layer_launch.csv python tools/layer_prof.py 4 8 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/layer_launch.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size') if 'Grid Size' in h else None
agg=collections.defaultdict(list)
for r in rows[1:]:
    agg[(r[ki][:40], r[gi] if gi else '')].append(float(r[vi].replace(',','')))
for k,v in agg.items(): print(f"{k[0]:40s} grid={k[1]:14s} n={len(v):3d} mean={sum(v)/len(v)/1000:.2f} us")
PY
