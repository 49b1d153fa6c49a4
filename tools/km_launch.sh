ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(assign|fixup|eps|update)" --csv --log-file gpurun_out/launch_km.csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu --max-iters 3 > /dev/null 2>&1
CKV_DEBUG_KMEANS=1 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > gpurun_out/dbg_km.json 2> gpurun_out/dbg_km.err
