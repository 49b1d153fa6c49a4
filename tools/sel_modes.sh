for m in ${MODES:-0 1}; do
CKV_SEL_MODE=$m ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_select|k_score" --csv --log-file gpurun_out/sel_mode$m.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu --max-iters 2 > /dev/null 2>&1
done
CKV_SELECT_UNFUSED=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_select|k_score" --csv --log-file gpurun_out/sel_unfused.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu --max-iters 2 > /dev/null 2>&1
