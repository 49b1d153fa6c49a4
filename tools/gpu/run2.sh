set -x
python -m pytest tests/test_gpu_bench_world.py -x -q 2>&1 | tail -5
CKV_TRACE_HOST=1 python tools/prefill_jitter.py 12 > gpurun_out/jitter.out 2> gpurun_out/jitter.err
tail -12 gpurun_out/jitter.out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
tail -c 1500 gpurun_out/bench_r2a.json; tail -3 gpurun_out/bench_r2a.err
