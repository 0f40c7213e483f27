"""Golden plan reports from the REAL reference CLI (``minishampoo plan``, cli.py:168-218).

Build container only (``/root/reference`` does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_plan_reports.py

Writes tests/golden/plan_reports.json: for each case, the CLI's flags and its stdout JSON.
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from minishampoo.cli import main  # noqa: E402

CASES = [
    ["--max-preconditioner-dim", "512"],
    ["--max-preconditioner-dim", "128", "--world-size", "4"],
    ["--max-preconditioner-dim", "64", "--world-size", "8", "--num-trainers-per-group", "2",
     "--steps", "7"],
    ["--max-preconditioner-dim", "256", "--world-size", "2", "--large-dim-method", "diagonal",
     "--hidden-widths", "300,100"],
    ["--max-preconditioner-dim", "100", "--world-size", "4", "--large-dim-method", "adagrad",
     "--hidden-widths", "1000"],
]


def run(flags):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = main(["plan", *flags])
    assert rc == 0, flags
    return json.loads(buf.getvalue())


if __name__ == "__main__":
    out = [{"flags": f, "report": run(f)} for f in CASES]
    with open(os.path.join(HERE, "plan_reports.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote", len(out), "plan reports")
