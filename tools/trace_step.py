"""Per-layer timeline of the CUDA-graph decode step from globaltimer stamps
(debug build path: KVC_K1_TRACE_PTR).  Kernel A: every warp's entry and exit;
kernel B: every CTA's dependency-wait release and exit.  Runs bench.py's state
(default B=64; pass bench flags, e.g. --batch 8) and prints, per layer, in us
relative to that layer's first kernel-A warp entry:
  A warps' exit p50 / p90 / max, B first release, B last exit, next layer's
  first A entry.
Usage: python tools/trace_step.py [bench flags]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.argv = [sys.argv[0]] + ["--no-cpu", "--no-e2e", "--no-fragmented", "--prefill-seqs", "2"] + sys.argv[1:]

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    buf = torch.zeros(64 * 65536, dtype=torch.int64, device=dev)
    os.environ["KVC_K1_TRACE_PTR"] = str(buf.data_ptr())
    import bench
    args = bench.parse()
    S = bench.build(args, dev, 0)
    bench.eviction_rounds(S, args)
    bench.populate(S, args)
    buf.zero_()
    bench.decode_bench(S, args)
    torch.cuda.synchronize()
    t = buf.view(64, 65536).cpu().numpy().astype(np.float64)
    L = min(args.layers, 64)
    rows = []
    for m in range(L):
        a = t[m, :32768].reshape(-1, 2)
        a = a[(a[:, 0] > 0) & (a[:, 1] > 0)]
        b = t[m, 32768:].reshape(-1, 2)
        b = b[(b[:, 0] > 0) & (b[:, 1] > 0)]
        if len(a) == 0:
            continue
        t0 = a[:, 0].min()
        ends = np.sort(a[:, 1] - t0) / 1e3
        nxt = None
        if m + 1 < L:
            a2 = t[m + 1, :32768].reshape(-1, 2)
            a2 = a2[(a2[:, 0] > 0)]
            if len(a2):
                nxt = (a2[:, 0].min() - t0) / 1e3
        rows.append((m, len(a), (a[:, 0].max() - t0) / 1e3, ends[len(ends) // 2], ends[int(len(ends) * 0.9)], ends[-1],
                     (b[:, 0].min() - t0) / 1e3 if len(b) else float("nan"),
                     (b[:, 1].max() - t0) / 1e3 if len(b) else float("nan"), nxt))
    print("layer warps A_entry_max A_exit_p50 A_exit_p90 A_exit_max B_release_first B_exit_last next_A_entry")
    for r in rows:
        print(" ".join(f"{x:.2f}" if isinstance(x, float) else str(x) for x in r))
    per = [r[8] for r in rows if r[8] is not None]
    if per:
        print(f"mean layer period {np.mean(per):.2f} us; mean A exit max {np.mean([r[5] for r in rows]):.2f}; "
              f"mean B exit {np.nanmean([r[7] for r in rows]):.2f}")


if __name__ == "__main__":
    main()
