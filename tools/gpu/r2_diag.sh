#!/bin/bash
# Diagnostics: prefill per-launch list (ncu), e2e split, host overhead.
O=gpurun_out
mkdir -p $O
timeout 600 python tools/e2e_breakdown.py > $O/e2e_breakdown.txt 2>&1; tail -2 $O/e2e_breakdown.txt
timeout 600 python tools/host_overhead.py 32768 > $O/host_overhead.txt 2>&1; tail -5 $O/host_overhead.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"k_assign|k_fixup|k_update|k_index|k_control|k_repair|k_scan|k_eps|k_compact|k_dirs|k_init|k_copy" \
    --csv --log-file $O/launch_prefill.csv python tools/prefill_jitter.py 1 > /dev/null 2>&1
python tools/launch_table.py $O/launch_prefill.csv 2>&1 | head -30
