#!/bin/bash
# full GPU suite + smoke + default bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
p=d.get('prefill',{})
print('value',round(d['value']),'ms/step',round(d['ms_per_step']*1000,1),'e2e',round(d['e2e']['value']),'attend frac',round(d['roofline']['frac'],3),'select us',round(d['kernels_us']['k_select'],1))
print('prefill',p.get('ms'),p.get('ms_all'),'frac',p.get('frac_of_bf16_peak'))
print('per_layer',d.get('per_layer',{}).get('ms_per_step'), 'clocks', d.get('clocks'))
PY
