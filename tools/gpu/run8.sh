for v in 0 1; do
  CKV_SEL_MODE=$v python bench.py --steps 30 --warmup 5 --no-extra --no-cpu > gpurun_out/b_sm_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/b_sm_$v.json').read().strip().splitlines()[-1])
print('selmode=$v', round(d['ms_per_step']*1e3,1), d['kernels_us'])"
done
ncu --set full --import-source on --clock-control none -k regex:k_select_fused -s 5 -c 1 -o gpurun_out/select_r2a python bench.py --steps 3 --warmup 3 --no-extra --no-cpu > /dev/null 2>&1
