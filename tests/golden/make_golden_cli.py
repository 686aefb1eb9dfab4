"""Golden stdout / exit codes of the REFERENCE CLI (cli.py) for the commands
this package mirrors (select, evaluate, cdf), made by running the reference
package in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cli.py

Writes cli_graph.txt (a weighted edge list with sparse original ids),
cli_seeds.txt and cli_cases.json: per case the argv (paths relative to this
directory, "{out}" for a scratch output file), the exit code, stdout, and
the --out file's text when one is written.  Timing lines go to stderr and are
not recorded.
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

from infmax.cli import main  # noqa: E402


def write_inputs():
    rng = np.random.default_rng(11)
    ids = rng.choice(np.arange(10, 100_000), size=900, replace=False)
    lines = ["# synthetic weighted edge list: u v w"]
    seen = set()
    while len(seen) < 4200:
        a, b = rng.integers(0, len(ids), size=2)
        if a == b or (a, b) in seen or (b, a) in seen:
            continue
        seen.add((a, b))
        lines.append(f"{ids[a]} {ids[b]} {rng.random() * 0.4:.6f}")
    (HERE / "cli_graph.txt").write_text("\n".join(lines) + "\n")
    seeds = [int(ids[i]) for i in (3, 17, 250, 600)]
    (HERE / "cli_seeds.txt").write_text("# seeds\n" + "\n".join(map(str, seeds)) + "\n")


CASES = [
    ["select", "--graph", "cli_graph.txt", "--k", "8", "--r", "256", "--seed", "3", "--threads", "1"],
    ["select", "--graph", "cli_graph.txt", "--k", "5", "--r", "100", "--weights", "file", "--threads", "1",
     "--out", "{out}"],
    ["select", "--graph", "cli_graph.txt", "--k", "12", "--r", "64", "--weights", "const:0.05", "--threads", "1"],
    ["select", "--graph", "cli_graph.txt", "--k", "3", "--r", "40", "--weights", "normal:0.1,0.05",
     "--seed", "9", "--threads", "1"],
    ["select", "--graph", "cli_graph.txt", "--k", "901", "--r", "8", "--threads", "1"],        # k > n: exit 3
    ["select", "--graph", "missing_graph.txt", "--k", "3", "--threads", "1"],                # I/O: exit 2
    ["evaluate", "--graph", "cli_graph.txt", "--seeds-file", "cli_seeds.txt", "--r-eval", "5000", "--seed", "4"],
    ["evaluate", "--graph", "cli_graph.txt", "--seeds-file", "cli_seeds.txt", "--weights", "file",
     "--r-eval", "300"],
    ["cdf", "--graph", "cli_graph.txt", "--r", "64", "--bins", "20"],
    ["cdf", "--graph", "cli_graph.txt", "--r", "32", "--bins", "10", "--weights", "uniform:0,0.3",
     "--out", "{out}"],
]


def run(argv):
    with tempfile.TemporaryDirectory() as tmp:
        out = os.path.join(tmp, "out.txt")
        args = [a.replace("{out}", out) for a in argv]
        buf = io.StringIO()
        cwd = os.getcwd()
        os.chdir(HERE)
        try:
            with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(io.StringIO()):
                code = main(args)
        finally:
            os.chdir(cwd)
        text = Path(out).read_text() if os.path.exists(out) else None
    return {"argv": argv, "code": code, "stdout": buf.getvalue(), "out_text": text}


if __name__ == "__main__":
    write_inputs()
    res = [run(a) for a in CASES]
    (HERE / "cli_cases.json").write_text(json.dumps(res, indent=1))
    for r in res:
        print(r["code"], " ".join(r["argv"][:3]), r["stdout"].splitlines()[:4], file=sys.stderr)
