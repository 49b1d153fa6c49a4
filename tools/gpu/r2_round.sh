#!/bin/bash
# Round-2 evidence pass (under gpurun): GPU suite, default bench line, ncu
# launch lists + one --set full capture each for decode and prefill, and the
# secondary config lines.  Summaries: tools/profile_summary.py r02_<x> ...
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
B="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu --no-extra"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_select|k_score|k_attend|k_append" \
    --csv --log-file $O/launch_decode.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_select_fused|k_attend" \
    --launch-skip 6 -c 2 -o $O/prof_decode -f $B > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"k_assign|k_fixup|k_update|k_index|k_control|k_repair|k_scan|k_eps|k_compact|k_dirs|k_init|k_copy" \
    --csv --log-file $O/launch_prefill.csv python tools/prefill_jitter.py 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_assign_tc2" --launch-skip 2 -c 1 \
    -o $O/prof_assign -f python tools/prefill_jitter.py 1 > /dev/null 2>&1
timeout 600 python bench.py --config A --steps 10 --warmup 3 > $O/cfgA.json 2> $O/cfgA.err
timeout 900 python bench.py --config C --steps 5 --warmup 3 > $O/cfgC.json 2> $O/cfgC.err
timeout 900 python bench.py --config E --steps 10 --warmup 3 > $O/cfgE.json 2> $O/cfgE.err
ls -la $O
