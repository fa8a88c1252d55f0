timeout 600 python -m pytest tests/test_gpu_compress.py tests/test_gpu_prefill_compress.py tests/test_gpu_engine.py -x -q -p no:cacheprovider 2>&1 | tail -2
for v in "KVC_COPY_U=8" "KVC_K3_SPLIT=1" "KVC_K4_UNFUSED=1"; do
  echo "== $v"
  env $v timeout 300 python tools/time_evict.py | python -c "import json,sys; r=json.load(sys.stdin); print('k34', [round(x['k34_ms'],4) for x in r if 'k34_ms' in x], 'k3', [round(x['k3_ms'],4) for x in r if 'k3_ms' in x], 'fused', [round(x['fused_prefill_compress_ms'],4) for x in r if 'fused_prefill_compress_ms' in x])"
done
