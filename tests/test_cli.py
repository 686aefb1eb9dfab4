"""The CLI front end (cli.py) against the reference CLI's own stdout and exit
codes (tests/golden/cli_cases.json, made by tests/golden/make_golden_cli.py
running the reference package)."""

import contextlib
import io
import json
import os

import pytest

from conftest import ROOT

GOLDEN = ROOT / "tests" / "golden"


def run_cli(argv, tmp_path):
    from paper_2008_03095_b200.cli import main
    out = str(tmp_path / "out.txt")
    args = [a.replace("{out}", out) for a in argv]
    buf = io.StringIO()
    cwd = os.getcwd()
    os.chdir(GOLDEN)
    try:
        with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(io.StringIO()):
            try:
                code = main(args)
            except SystemExit as e:        # argparse usage errors
                code = e.code
    finally:
        os.chdir(cwd)
    text = open(out).read() if os.path.exists(out) else None
    return code, buf.getvalue(), text


@pytest.mark.parametrize("argv", [
    [],
    ["bench", "--config", "x.ini"],                                   # not offered: checker harness
    ["select", "--graph", "cli_graph.txt", "--k", "3", "--algo", "mixgreedy"],
    ["select", "--graph", "cli_graph.txt", "--k", "3", "--weights", "bogus:1"],
    ["select", "--graph", "cli_graph.txt"],                           # --k missing
])
def test_usage_errors_exit_1(argv, tmp_path):
    code, out, _ = run_cli(argv, tmp_path)
    assert code == 1 and out == ""


def test_unreadable_graph_exits_2(tmp_path):
    code, out, _ = run_cli(["select", "--graph", "missing_graph.txt", "--k", "3"], tmp_path)
    assert code == 2 and out == ""


CASES = json.loads((GOLDEN / "cli_cases.json").read_text())


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[" ".join(c["argv"][:1] + c["argv"][3:7]) for c in CASES])
def test_cli_matches_reference_output(case, tmp_path):
    code, out, text = run_cli(case["argv"], tmp_path)
    assert code == case["code"]
    assert out == case["stdout"]
    assert text == case["out_text"]
