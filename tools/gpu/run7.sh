ncu --set full --import-source on --clock-control none -k regex:k_assign_tc -s 10 -c 1 -o gpurun_out/assign_r2b python tools/prefill_jitter.py 1 > /dev/null 2>&1
ls -la gpurun_out/assign_r2b.ncu-rep
