# compute-sanitizer memcheck over the GPU test files named on the command line
O=gpurun_out
for t in "$@"; do
  timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/$t.py -x -q > $O/san_$t.txt 2>&1
  echo "memcheck $t: $(grep 'ERROR SUMMARY' $O/san_$t.txt | tail -1) $(tail -1 $O/san_$t.txt)"
done
