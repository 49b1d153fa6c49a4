#!/bin/bash
for p in 0 3; do
CKV_KM_PERM_AT=$p timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none \
    -k regex:"k_assign|k_fixup|k_update|k_index|k_permute" --csv --log-file gpurun_out/perm$p.csv python tools/prefill_jitter.py 1 > /dev/null 2>&1
python - <<PY
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/perm$p.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); mi=h.index('Metric Name')
agg=collections.defaultdict(lambda:[0.0,0.0])
for r in rows[1:]:
    k=r[ki].split('(')[0][:30]
    if r[mi]=='gpu__time_duration.sum': agg[k][0]+=float(r[vi].replace(',',''))
    else: agg[k][1]+=float(r[vi].replace(',',''))
print("perm_at $p:", "  ".join(f"{k} {t/1e6:.2f}ms {n/1e6:.0f}Mi" for k,(t,n) in sorted(agg.items(), key=lambda x:-x[1][0])[:5]))
PY
done
