python bench.py --config D --steps 5 --warmup 3 > gpurun_out/cfgD.json 2> gpurun_out/cfgD.err
python -c "
import json; d=json.loads(open('gpurun_out/cfgD.json').read().strip().splitlines()[-1])
for k,v in d.items():
  if k.startswith('R'): print(k, {x: v[x] for x in ('hit_rate','step_us_mean','step_us_plain','clustering_us_per_event','tokens_per_s') }, v.get('tier'))
"
tail -3 gpurun_out/cfgD.err
