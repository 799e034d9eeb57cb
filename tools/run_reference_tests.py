"""Run the reference's own test suite (latquad, /root/reference/pkg/tests)
unmodified against this repo's GPU package, through the import shim
tools/refcompat/latquad.

    python tools/run_reference_tests.py stage    # build container: copy the tests
                                                 # into build/reftests (git-ignored,
                                                 # never committed; travels with gpurun)
    python tools/run_reference_tests.py run      # GPU box: pytest them, write
                                                 # gpurun_out/reftests.json
    python tools/run_reference_tests.py clean    # delete the staged copy

The staged copy exists only for the run; the summary (per-test outcome and
the first line of each failure) is what gets committed, under profiles/.
"""

import json
import os
import shutil
import subprocess
import sys
import xml.etree.ElementTree as ET

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg/tests"
STAGE = os.path.join(REPO, "build", "reftests")
OUT = os.path.join(REPO, "gpurun_out")


def stage():
    shutil.rmtree(STAGE, ignore_errors=True)
    shutil.copytree(SRC, STAGE)
    for root, _, files in os.walk(STAGE):
        for f in files:
            os.chmod(os.path.join(root, f), 0o644)
    print(f"staged {len(os.listdir(STAGE))} files into {STAGE}")


def run(extra=()):
    os.makedirs(OUT, exist_ok=True)
    xml = os.path.join(OUT, "reftests.xml")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(REPO, "tools", "refcompat"), REPO]),
               PYTHONDONTWRITEBYTECODE="1")
    # latquad.plots (matplotlib figures, out of scope) is a stub in the shim
    cmd = [sys.executable, "-m", "pytest", STAGE, "-q", "-p", "no:cacheprovider", "--timeout", "600",
           f"--junitxml={xml}", "-o", "junit_family=xunit1",
           "--rootdir", STAGE, *extra]
    rc = subprocess.call(cmd, env=env, cwd=STAGE)
    cases = []
    for tc in ET.parse(xml).getroot().iter("testcase"):
        outcome, msg = "passed", ""
        for tag in ("failure", "error", "skipped"):
            el = tc.find(tag)
            if el is not None:
                outcome = {"failure": "failed", "error": "error", "skipped": "skipped"}[tag]
                msg = (el.get("message") or "").strip().splitlines()[0][:300] if el.get("message") else ""
                break
        cases.append({"test": f"{tc.get('classname')}::{tc.get('name')}", "outcome": outcome, "message": msg})
    counts = {}
    for c in cases:
        counts[c["outcome"]] = counts.get(c["outcome"], 0) + 1
    with open(os.path.join(OUT, "reftests.json"), "w") as fh:
        json.dump({"pytest_rc": rc, "counts": counts, "cases": cases}, fh, indent=1)
    print(json.dumps(counts))
    return rc


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "run"
    if what == "stage":
        stage()
    elif what == "clean":
        shutil.rmtree(STAGE, ignore_errors=True)
    else:
        run(sys.argv[2:])
