for m in ${MODES:-0 1 2}; do
CKV_TC_MODE=$m ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_assign_tc" --csv --log-file gpurun_out/tc_mode$m.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu --no-extra --max-iters 2 > /dev/null 2>&1
done
