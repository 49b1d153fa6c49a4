#!/bin/bash
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"k_assign|k_fixup|k_update|k_index|k_control|k_repair|k_scan|k_eps|k_compact|k_dirs|k_init|k_copy|k_validate|k_fill|k_set" \
    --csv --log-file gpurun_out/launch_prefill.csv python tools/prefill_jitter.py 1 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/launch_prefill.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows[1:]:
    k=r[ki].split('(')[0][:40]; agg[k][0]+=1; agg[k][1]+=float(r[vi].replace(',',''))
tot=sum(v[1] for v in agg.values())
for k,(n,t) in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{k:40s} n={n:5d} total={t/1e6:8.2f} ms  {100*t/tot:5.1f}%")
print("total", tot/1e6, "ms")
PY
