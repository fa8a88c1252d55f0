ROUNDS=3 timeout 600 python tools/time_decode_round.py 2>/dev/null | tail -1
ROUNDS=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"k_load|k_hist|k_bounds|k_select|k_offsets|k_compact_warp|k_copy_kv|k_free_total" --csv --log-file gpurun_out/dr.csv python tools/time_decode_round.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/dr.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size')
for r in rows[1:]: print(r[ki].split('(')[0][-28:], r[gi], float(r[vi])/1e3)
PY
