python tools/decode_batch_prof.py 6
ncu --set full --import-source on --clock-control none -k regex:k_kmeans_small -s 2 -c 1 -o gpurun_out/kmsmall python tools/decode_batch_prof.py 4 > gpurun_out/kmsmall_ncu.log 2>&1
tail -3 gpurun_out/kmsmall_ncu.log
