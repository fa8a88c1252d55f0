ncu --set full --clock-control none --import-source on -k regex:"k_load|k_hist|k_bounds|k_compact16|k_copy_published" -s 12 -c 6 -o gpurun_out/prof_k34_r2 python tools/time_evict.py > gpurun_out/p34.log 2>&1
tail -3 gpurun_out/p34.log
