for v in "" "KVC_K4_UNFUSED=1"; do
  echo "== $v"
  env $v timeout 300 python tools/time_evict.py | python -c "import json,sys; r=json.load(sys.stdin); print('k34', [round(x['k34_ms'],4) for x in r if 'k34_ms' in x], 'k3', [round(x['k3_ms'],4) for x in r if 'k3_ms' in x], 'fused', [round(x['fused_prefill_compress_ms'],4) for x in r if 'fused_prefill_compress_ms' in x], 'host', [round(x['host_enqueue_ms'],3) for x in r if 'k34_ms' in x])"
  env $v KVC_K4_TRACE=1 timeout 300 python tools/time_evict.py 2>&1 | grep "k4 trace" | head -4
done
