"""Run the reference's own test files against paper_2207_11620_b200.

    python tools/run_reference_tests.py --fetch          # here: copy /root/reference/pkg/tests
    python tools/run_reference_tests.py --run TAG        # GPU box: run them -> gpurun_out/reftests_TAG/ (copied to profiles/)

--fetch copies the test files (read-only reference, not committed: tools/refshim/_tests
is git-ignored but travels to the GPU box with the snapshot).  --run executes each
file with `neuralvol` resolved to tools/refshim/neuralvol (module aliases onto this
package + the numba FFI served by the C ABI) and the one numpy adapter of
tools/refshim/refshim_adapter.py, and records pass / fail / error per test.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys
import xml.etree.ElementTree as ET
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SHIM = ROOT / "tools" / "refshim"
DST = SHIM / "_tests"
FILES = ["test_encoding.py", "test_network.py", "test_trainer.py", "test_sampler.py", "test_macrocell.py",
         "test_render.py", "test_volume.py", "test_camera.py", "test_estimator.py", "test_acceptance.py"]


def fetch():
    src = Path("/root/reference/pkg/tests")
    DST.mkdir(parents=True, exist_ok=True)
    for f in ["conftest.py"] + FILES:
        shutil.copy(src / f, DST / f)
    print("copied", len(FILES) + 1, "files to", DST)


def run(tag: str):
    out = ROOT / "gpurun_out" / f"reftests_{tag}"
    out.mkdir(parents=True, exist_ok=True)
    env = dict(os.environ, PYTHONPATH=f"{SHIM}:{ROOT}:" + os.environ.get("PYTHONPATH", ""))
    rows, totals = [], {"passed": 0, "failed": 0, "error": 0, "skipped": 0}
    for f in FILES:
        xml = out / (f + ".xml")
        cmd = [sys.executable, "-m", "pytest", str(DST / f), "-q", "-p", "refshim_adapter", "-p", "no:cacheprovider",
               "--timeout", "900", f"--junitxml={xml}", "--rootdir", str(DST)]
        r = subprocess.run(cmd, env=env, cwd=str(DST), capture_output=True, text=True, timeout=3600)
        (out / (f + ".log")).write_text(r.stdout[-20000:] + r.stderr[-5000:])
        if not xml.exists():
            rows.append({"file": f, "test": "<collection>", "outcome": "error", "detail": r.stdout[-400:]})
            totals["error"] += 1
            continue
        for tc in ET.parse(xml).getroot().iter("testcase"):
            name = tc.get("name")
            outcome, detail = "passed", ""
            for k in ("failure", "error", "skipped"):
                e = tc.find(k)
                if e is not None:
                    outcome = {"failure": "failed", "error": "error", "skipped": "skipped"}[k]
                    detail = (e.get("message") or "")[:300]
            totals[outcome] += 1
            rows.append({"file": f, "test": name, "outcome": outcome, "detail": detail})
    res = {"tag": tag, "totals": totals, "tests": rows,
           "how": "reference test files run unmodified; `neuralvol` -> tools/refshim (aliases onto "
                  "paper_2207_11620_b200 + the numba FFI over the C ABI); adapter (tools/refshim/refshim_adapter.py): "
                  "numpy reads CUDA tensors, numpy/list values assign into CUDA tensors, Tensor.copy = clone, Tensor.astype -> numpy"}
    (out / f"reference_tests_{tag}.json").write_text(json.dumps(res, indent=1))
    lines = [f"# Reference test files against paper_2207_11620_b200 ({tag})", "",
             f"Totals: {totals}", "", "| file | test | outcome | detail |", "|---|---|---|---|"]
    for r in rows:
        d = r["detail"].replace("|", "/").replace("\n", " ")[:160]
        lines.append(f"| {r['file']} | {r['test']} | {r['outcome']} | {d} |")
    (out / f"reference_tests_{tag}.md").write_text("\n".join(lines) + "\n")
    print(json.dumps(totals))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--fetch", action="store_true")
    ap.add_argument("--run")
    a = ap.parse_args()
    if a.fetch:
        fetch()
    if a.run:
        run(a.run)
