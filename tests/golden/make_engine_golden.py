"""Run the REFERENCE engine (pagedkv, /root/reference) on the workloads of
engine_workload.py and store its StepRecords as golden fixtures
(tests/golden/engine_cases.json).  Run in the build container only:
    python tests/golden/make_engine_golden.py
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

import pagedkv as R  # noqa: E402
import pagedkv.engine as RE  # noqa: E402
from engine_workload import CASES, SHAPE, SHARD_WORLD, HashTokens, make_policy, shard  # noqa: E402


def run(kw, indexed_reqs):
    cfg = R.AttentionConfig(SHAPE["n_q"], SHAPE["n_k"], SHAPE["d"], SHAPE["layers"])
    eng = RE.Engine(cfg, R.MetricConfig(), make_policy(RE, kw["policy"]), kw["num_blocks"], SHAPE["block_size"],
                    rate=kw["rate"], budget_floor=kw["budget_floor"], record_schedules=True)
    for i, (pl, ot) in indexed_reqs:
        eng.submit(HashTokens(1000 + i, pl, ot, SHAPE["layers"], SHAPE["n_q"], SHAPE["n_k"], SHAPE["d"]))
    return [r.to_dict() for r in eng.run_to_completion()]


def main():
    out = []
    for name, kw, reqs in CASES:
        recs = run(kw, list(enumerate(reqs)))
        # the same workload sharded over SHARD_WORLD ranks: each rank's own
        # engine (own pool of num_blocks) over the requests it owns
        shards = [run(kw, shard(reqs, rank)) for rank in range(SHARD_WORLD)]
        out.append({"name": name, "records": recs, "shards": shards})
        print(name, len(recs), "steps", sum(r["preemptions"] for r in recs), "preemptions",
              sum(r["compressions"] for r in recs), "compressions; shard steps", [len(x) for x in shards])
    with open(os.path.join(HERE, "engine_cases.json"), "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
