#!/bin/bash
# BASELINE.json configs and the decode batch sweep through bench.py (one GPU),
# one JSON line each under gpurun_out/configs/.  Run from the repo root.
mkdir -p gpurun_out/configs
run() {
  local name=$1; shift
  timeout 900 python bench.py --no-cpu --no-e2e --no-fragmented "$@" > gpurun_out/configs/$name.json 2> gpurun_out/configs/$name.err
  echo "$name rc=$?"
}
run toy --preset toy --prefill-seqs 2
# Mistral-7B shapes over the LongBench-like 8k-32k prompt range, 16x
for L in 8192 16384 32768; do run m7b_b64_L$L --preset m7b --context $L --prefill-seqs 2; done
run l70b_b64 --preset l70b --prefill-seqs 2
# batch sweep at 32k: 8x (the headline rate), 1x (no eviction) and 32x
for b in 1 8 32 64 128 192 256; do run l8b_b$b --batch $b --prefill-seqs 2; done
for b in 1 8 32; do run l8b_b${b}_r1 --batch $b --rate 1 --prefill-seqs 2; done
for b in 8 64 256 512; do run l8b_b${b}_r32 --batch $b --rate 32 --prefill-seqs 2; done
