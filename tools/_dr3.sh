timeout 900 python -m pytest tests/test_gpu_compress.py tests/test_gpu_engine.py -x -q -p no:cacheprovider 2>&1 | tail -1
ROUNDS=3 timeout 600 python tools/time_decode_round.py 2>/dev/null | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('round', [round(x,4) for x in r['ms']])"
timeout 300 python tools/time_evict.py | python -c "import json,sys; r=json.load(sys.stdin); print('k34', [round(x['k34_ms'],4) for x in r if 'k34_ms' in x][1:], 'k3', [round(x['k3_ms'],4) for x in r if 'k3_ms' in x][1:])"
