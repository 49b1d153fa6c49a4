#!/bin/bash
# Closing evidence of the last round-2 session: the round pass (GPU suite,
# default bench line, ncu launch lists + --set full captures, configs A/C/E),
# smoke, the reference arm, and a memcheck pass over the changed paths.
O=gpurun_out
mkdir -p $O
bash tools/gpu/r2_round.sh
timeout 300 python __graft_entry__.py --smoke > $O/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
for t in test_gpu_session test_gpu_kmeans_tc; do
  timeout 1200 compute-sanitizer --tool memcheck python -m pytest tests/$t.py -x -q > $O/san_$t.txt 2>&1
  echo "memcheck $t: $(grep 'ERROR SUMMARY' $O/san_$t.txt | tail -1) $(tail -1 $O/san_$t.txt)"
done
