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
from engine_workload import CASES, SHAPE, HashTokens  # noqa: E402


def main():
    out = []
    for name, kw, reqs in CASES:
        cfg = R.AttentionConfig(SHAPE["n_q"], SHAPE["n_k"], SHAPE["d"], SHAPE["layers"])
        eng = RE.Engine(cfg, R.MetricConfig(), RE.POLICY_PRESETS[kw["policy"]], kw["num_blocks"], SHAPE["block_size"],
                       rate=kw["rate"], budget_floor=kw["budget_floor"], record_schedules=True)
        for i, (pl, ot) in enumerate(reqs):
            eng.submit(HashTokens(1000 + i, pl, ot, SHAPE["layers"], SHAPE["n_q"], SHAPE["n_k"], SHAPE["d"]))
        recs = [r.to_dict() for r in eng.run_to_completion()]
        out.append({"name": name, "records": recs})
        print(name, len(recs), "steps", sum(r["preemptions"] for r in recs), "preemptions",
              sum(r["compressions"] for r in recs), "compressions")
    with open(os.path.join(HERE, "engine_cases.json"), "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
