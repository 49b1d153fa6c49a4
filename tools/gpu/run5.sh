python tools/prefill_jitter.py 12 > gpurun_out/jitter2.out 2>&1; tail -12 gpurun_out/jitter2.out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r2b.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step", "kernels_us", "e2e")})
print(d["prefill"])
print({k: d["config_D"][k] for k in d["config_D"] if k.startswith("R")})
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prefill_launches_r2.csv python tools/prefill_jitter.py 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_assign_tc -s 10 -c 1 -o gpurun_out/assign_r2a python tools/prefill_jitter.py 1 > /dev/null 2>&1
ls gpurun_out
