#!/bin/bash
# BASELINE.json configs and the decode batch sweep through bench.py (one GPU),
# one JSON line each under gpurun_out/configs/.  Run from the repo root.
mkdir -p gpurun_out/configs
run() {
  local name=$1; shift
  timeout 900 python bench.py --no-cpu --no-e2e "$@" > gpurun_out/configs/$name.json 2> gpurun_out/configs/$name.err
  echo "$name rc=$?"
}
run toy --preset toy --prefill-seqs 2
run m7b_b64 --preset m7b
run l70b_b64 --preset l70b --prefill-seqs 2
for b in 1 8 32 64 128 192 256; do run l8b_b$b --batch $b --prefill-seqs 2; done
run l8b_b16_r1 --batch 16 --rate 1 --prefill-seqs 2
run l8b_b256_r32 --batch 256 --rate 32 --prefill-seqs 2
run l8b_b512_r32 --batch 512 --rate 32 --prefill-seqs 2
