"""Run the reference's own test suite (pkg/tests) against the B200 package
through an import swap: `pagedkv` resolves to tools/refsuite/pagedkv, which
re-exports paper_2410_00161_b200.  Test infrastructure only.

Here (where /root/reference exists) the tests are copied into the git-ignored
baseline/_ref/tests, which travels to the GPU box; run this script there:
    python tools/run_reference_suite.py            # -> profiles/r2_reference_suite.json
"""
import json
import os
import shutil
import subprocess
import sys
import xml.etree.ElementTree as ET

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DST = os.path.join(ROOT, "baseline", "_ref", "tests")
SRC = "/root/reference/pkg/tests"


def main():
    if os.path.isdir(SRC):
        shutil.rmtree(DST, ignore_errors=True)
        shutil.copytree(SRC, DST)
    if "--copy-only" in sys.argv:
        return
    xml = os.path.join(ROOT, "gpurun_out", "refsuite.xml")
    if "--parse-only" not in sys.argv:
        run(xml)
    summarize(xml)


def run(xml):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tools", "refsuite"), ROOT, DST])
    os.makedirs(os.path.dirname(xml), exist_ok=True)
    subprocess.run([sys.executable, "-m", "pytest", DST, "-q", "-p", "no:cacheprovider", "--junitxml", xml,
                    "--continue-on-collection-errors",
                    "-o", "addopts="], env=env, cwd=DST)


def summarize(xml):
    res = {}
    for case in ET.parse(xml).getroot().iter("testcase"):
        f = case.get("classname", "").split(".")[0] or case.get("name", "?")
        r = res.setdefault(f, {"passed": 0, "failed": 0, "error": 0, "skipped": 0, "first_failures": []})
        kids = [c.tag for c in case]
        if "failure" in kids or "error" in kids:
            key = "failed" if "failure" in kids else "error"
            r[key] += 1
            if len(r["first_failures"]) < 4:
                el = case.find("failure" if key == "failed" else "error")
                r["first_failures"].append(f"{case.get('name')}: {(el.get('message') or '')[:160]}")
        elif "skipped" in kids:
            r["skipped"] += 1
        else:
            r["passed"] += 1
    tot = {k: sum(v[k] for v in res.values()) for k in ("passed", "failed", "error", "skipped")}
    out = {"what": "reference pkg/tests run with `pagedkv` imported from the B200 package (import swap)",
           "totals": tot, "per_file": res}
    with open(os.path.join(ROOT, "profiles", "r2_reference_suite.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(tot))


if __name__ == "__main__":
    main()
