# compute-sanitizer racecheck over the GPU test files named on the command line
O=gpurun_out
for t in "$@"; do
  timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/$t.py -x -q > $O/race_$t.txt 2>&1
  echo "race $t: $(grep 'RACECHECK SUMMARY' $O/race_$t.txt | tail -1) $(tail -1 $O/race_$t.txt)"
done
