#!/bin/bash
# Round-2 closing evidence pass: the round pass (GPU suite, default bench,
# ncu launch lists + --set full captures, configs A / C / E) and a sanitizer
# pass over the kernels changed since the last one.
O=gpurun_out
mkdir -p $O
bash tools/gpu/r2_round.sh
for t in test_gpu_select test_gpu_session test_gpu_headline; do
  timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/$t.py -x -q > $O/san_$t.txt 2>&1
  echo "memcheck $t: $(grep 'ERROR SUMMARY' $O/san_$t.txt | tail -1) $(tail -1 $O/san_$t.txt)"
done
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_select.py -x -q > $O/race_select.txt 2>&1
echo "racecheck select: $(grep -E 'RACECHECK SUMMARY|hazard' $O/race_select.txt | tail -1) $(tail -1 $O/race_select.txt)"
