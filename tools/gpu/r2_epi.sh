#!/bin/bash
# assignment epilogue budget: producer+MMA only (mode 2), loads only (mode 1), full (0);
# and the cluster-major operand from pass 3 on (CKV_KM_PERM_AT=3) on the full prefill
mkdir -p gpurun_out
MODES="0 1 2" bash tools/tc_modes.sh
for m in 0 1 2; do python tools/launch_table.py gpurun_out/tc_mode$m.csv | head -2 | sed "s/^/mode$m /"; done
timeout 300 python tools/prefill_jitter.py 5 2>/dev/null | tail -2
CKV_KM_PERM_AT=3 timeout 300 python tools/prefill_jitter.py 5 2>/dev/null | tail -2
CKV_KM_PERM_AT=3 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_assign_tc2" \
    --csv --log-file gpurun_out/perm_launch.csv python tools/prefill_jitter.py 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/perm_launch.csv')) if r]
h=None; v=[]
for r in rows:
    if 'Kernel Name' in r: h=r; continue
    if h and len(r)==len(h) and r[h.index('Metric Name')]=='gpu__time_duration.sum': v.append(round(float(r[h.index('Metric Value')].replace(',',''))/1000))
print('perm_at3 k_assign_tc2 per launch', v)
PY
