"""Round reports: emitReport csv | json (CPU).

build/report_test emits fixed RoundReports through include/hetm_b200/engine.hpp
emitReport: deterministic field order, one row per round plus a summary block,
identical values in both formats, summary throughput = sum committed / sum time,
an io-error on an unwritable path.
"""
import csv
import io
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIELDS = ["roundId", "outcome", "txCommittedHost", "txCommittedDev", "txWastedDev", "bytesLogs", "bytesMerge",
          "readOnlyHost", "cutShort", "devBatches", "execMs", "validateMs", "mergeMs"]


def test_emit_report_csv_json(tmp_path):
    exe = os.path.join(ROOT, "build", "report_test")
    if not os.path.exists(exe):
        pytest.skip("build/report_test not built (run __graft_entry__.build())")
    prefix = str(tmp_path / "rep")
    out = subprocess.run([exe, prefix], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stdout + out.stderr
    text = open(prefix + ".csv").read()
    rows_part, summary_part = text.split("\n\n")
    rows = list(csv.DictReader(io.StringIO(rows_part)))
    summary = next(csv.DictReader(io.StringIO(summary_part)))
    assert list(rows[0].keys()) == FIELDS                       # deterministic field order
    js = json.loads(open(prefix + ".json").read())
    assert [list(r.keys()) for r in js["rounds"]] == [FIELDS] * 3
    for c, j in zip(rows, js["rounds"]):                         # identical values
        for k in FIELDS:
            if k == "outcome":
                assert c[k] == j[k]
            else:
                assert float(c[k]) == float(j[k]), k
    assert [r["outcome"] for r in rows] == ["Commit", "DeviceAborted", "HostAborted"]
    # aborted sides count as wasted / zero committed
    assert rows[1]["txCommittedDev"] == "0" and rows[1]["txWastedDev"] == "4095"
    assert rows[2]["txCommittedHost"] == "0"
    # summary recomputed from the per-round rows
    committed = sum(int(r["txCommittedHost"]) + int(r["txCommittedDev"]) for r in rows)
    t_ms = sum(float(r["execMs"]) + float(r["validateMs"]) + float(r["mergeMs"]) for r in rows)
    assert int(summary["rounds"]) == 3 and float(summary["timeMs"]) == pytest.approx(t_ms, abs=1e-9)
    assert float(summary["throughputTxPerS"]) == pytest.approx(committed / (t_ms * 1e-3), abs=0.1)
    assert {k: float(v) for k, v in summary.items()} == {k: float(v) for k, v in js["summary"].items()}
