#!/bin/bash
# Profiling pass of one round (run under gpurun; reports land in gpurun_out/,
# summaries go to profiles/ via tools/profile_summary.py on this side).
#   decode (config B): launch list + one --set full capture of select / attend
#   prefill (config B): launch list of the k-means kernels + one k_assign_tc capture
#   config E step: launch list of the sharded decode kernels
set -x
O=gpurun_out
B="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu --no-extra"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_select|k_score|k_attend|k_append" \
    --csv --log-file $O/launch_decode.csv $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_select_fused|k_attend" \
    --launch-skip 6 -c 2 -o $O/prof_decode -f $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"k_assign|k_fixup|k_update|k_index|k_control|k_repair|k_scan|k_eps|k_compact|k_dirs|k_init|k_copy" \
    --csv --log-file $O/launch_prefill.csv $B --max-iters 50 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_assign_tc" --launch-skip 20 -c 1 \
    -o $O/prof_assign -f $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"k_score_range|k_select_scored|k_select_approx|k_attend|k_lse_merge|k_fill" \
    --csv --log-file $O/launch_cfgE.csv python bench.py --config E --steps 3 --warmup 2 > /dev/null 2>&1
ls -la $O
