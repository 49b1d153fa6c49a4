timeout 900 python -m pytest tests/test_gpu_session.py tests/test_gpu_headline.py tests/test_gpu_attend.py tests/test_gpu_sharded_decode.py -x -q 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 --no-extra --no-cpu > gpurun_out/b_pl.json 2>gpurun_out/b_pl.err
python -c "
import json; d=json.loads(open('gpurun_out/b_pl.json').read().strip().splitlines()[-1])
print(round(d['ms_per_step']*1e3,1), d['kernels_us'], d['per_layer'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pl_launches.csv python bench.py --steps 3 --warmup 3 --no-extra --no-cpu --e2e-steps 1 > /dev/null 2>&1
