for B in 8 32; do
for v in 256 512 1024; do
  KVC_K1_METRIC_DIV=$v timeout 600 python bench.py --batch $B --steps 20 --warmup 5 --no-cpu --no-e2e --no-fragmented --prefill-seqs 2 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B=$B mdiv=$v', round(r['ms_per_step'],4), 'ms/step', round(r['roofline']['frac'],3))"
done
done
for ib in 4 2 1; do
  KVC_K1_ITEM_BLOCKS=$ib timeout 600 python bench.py --batch 1 --steps 20 --warmup 5 --no-cpu --no-e2e --no-fragmented --prefill-seqs 2 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('B=1 ib=$ib', round(r['ms_per_step'],4), 'ms/step', round(r['roofline']['frac'],3))"
done
