"""Time the every-step policy's compression round alone: bench.py's default
state (Llama-8B shapes, B=64 x 32k, 8x), decode steps, then one compress()
over all 64 sequences (K3/K4 short-head path), a few rounds.
Usage: python tools/time_decode_round.py [rounds]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.argv = [sys.argv[0]] + ["--no-cpu", "--no-e2e", "--no-fragmented", "--prefill-seqs", "2"] + sys.argv[1:]

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    args = bench.parse()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    S = bench.build(args, dev, 0)
    bench.eviction_rounds(S, args)
    bench.populate(S, args)
    out = bench.decode_compression_rounds(S, args, rounds=int(os.environ.get("ROUNDS", "3")))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
