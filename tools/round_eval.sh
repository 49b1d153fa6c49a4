#!/bin/bash
# End-of-milestone evaluation under gpurun: full GPU tests, smoke, the default
# bench line, the reference arm, configs C / D / E, and the ncu evidence.
O=gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/eval_tests.txt
python __graft_entry__.py --smoke > $O/eval_smoke.txt 2>&1
python bench.py > $O/eval_bench.json 2> $O/eval_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/eval_bench_ref.json 2> $O/eval_bench_ref.err
python bench.py --config C --steps 10 --warmup 3 > $O/eval_cfgC.json 2> $O/eval_cfgC.err
python bench.py --config D > $O/eval_cfgD.json 2> $O/eval_cfgD.err
python bench.py --config E --steps 10 --warmup 3 > $O/eval_cfgE.json 2> $O/eval_cfgE.err
python bench.py --config A > $O/eval_cfgA.json 2> $O/eval_cfgA.err
B="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu --no-extra"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_select|k_score|k_attend|k_append" \
    --csv --log-file $O/launch_decode.csv $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_select_fused|k_attend" \
    --launch-skip 6 -c 2 -o $O/prof_decode -f $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"k_assign|k_fixup|k_update|k_index|k_control|k_repair|k_scan|k_eps|k_compact|k_dirs|k_init|k_copy" \
    --csv --log-file $O/launch_prefill.csv $B > /dev/null 2>&1
cat $O/eval_tests.txt $O/eval_smoke.txt
