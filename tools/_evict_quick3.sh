timeout 900 python -m pytest tests/test_gpu_compress.py tests/test_gpu_prefill_compress.py -x -q -p no:cacheprovider 2>&1 | tail -1
KVC_K4_TRACE=1 timeout 300 python tools/time_evict.py 2>&1 | grep "k4 trace" | sed -n 2,3p
for i in 1 2; do timeout 300 python tools/time_evict.py | python -c "import json,sys; r=json.load(sys.stdin); print('k34', [round(x['k34_ms'],4) for x in r if 'k34_ms' in x][1:], 'k3', [round(x['k3_ms'],4) for x in r if 'k3_ms' in x][1:])"; done
