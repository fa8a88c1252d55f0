#!/bin/bash
# Round capture on the GPU box (run under gpurun from the repo root):
#   launch list of the default bench, ncu --set full of K1, K2, K3/K4 and the
#   prefill kernels.  Summarise here with profiles/summarize.py.
set -x
O=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/b_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_decode_stream|k_decode_finish|k_decode_metric" -s 96 -c 3 \
    -o $O/prof_k1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $O/p1.log 2>&1
K2_LAYERS=32 ncu --set full --clock-control none --import-source on -k regex:k_window_persist -s 1 -c 1 \
    -o $O/prof_k2 python tools/time_k2.py > $O/p2.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_load|k_hist|k_compact16|k_copy_published|k_place_prompt_kv" -s 16 -c 16 \
    -o $O/prof_k34 python tools/time_evict.py > $O/p3.log 2>&1
ncu --set full --clock-control none -k regex:k_write_prefill -s 1 -c 1 -o $O/prof_scatter python tools/time_scatter.py > $O/p4.log 2>&1
ls -la $O
