"""quantc CLI end to end on the committed small_cnn fixture:
calibrate -> search -> realize -> eval, file-mediated, deterministic."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(REPO, "paper_2103_14949_b200", "quantc")
FX = os.path.join(REPO, "tests", "fixtures", "quantc")
M = os.path.join(FX, "small_cnn.json")
S = os.path.join(FX, "specs", "int8_int32.json")
D = os.path.join(FX, "small_cnn_calibration.json")
E = os.path.join(FX, "small_cnn_evaluation.json")


def _run(*args):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return r.stdout


def test_cli_pipeline(b200, tmp_path):
    out = _run("calibrate", "-m", M, "-s", S, "-d", D, "--method", "kl", "--kl-bits", 8,
               "-o", tmp_path / "stats.json")
    stats = json.load(open(tmp_path / "stats.json"))
    g = b200.load_graph(M)
    spec = b200.parse_spec(open(S).read())
    edges = b200.simulated_edge_indices(g, b200.generate_topology(g, spec))
    lines = [ln for ln in out.splitlines()[1:] if ln.strip()]
    assert len(lines) == len(edges)
    assert "graph_fingerprint" in json.dumps(stats)
    for k in (1, 2):
        _run("search", "-m", M, "-s", S, "-d", D, "--stats", tmp_path / "stats.json",
             "--threshold", "max", "--method", "greedy", "--tol", 0.01,
             "-o", tmp_path / f"strategy{k}.json", "--trace", tmp_path / "trace.jsonl")
    a = open(tmp_path / "strategy1.json", "rb").read()
    assert a == open(tmp_path / "strategy2.json", "rb").read()  # deterministic
    strat = json.loads(a)
    bits = [v["bit"] for k, v in strat["edges"].items()] if "edges" in strat else \
        [v["bit"] for k, v in strat.items() if isinstance(v, dict) and "bit" in v]
    assert bits and all(4 <= b <= 8 for b in bits)
    _run("realize", "-m", M, "-s", S, "--strategy", tmp_path / "strategy1.json",
         "-o", tmp_path / "realized.json")
    out = _run("eval", "-a", M, "-b", M, "-d", E)
    assert "top1 agreement 1.000000" in out
    out = _run("eval", "-a", M, "-b", tmp_path / "realized.json", "-d", E)
    assert "top1 agreement" in out
    # a dataset the stats were not collected on is rejected (exit 2)
    r = subprocess.run([CLI, "search", "-m", M, "-s", S, "-d", E, "--stats",
                        str(tmp_path / "stats.json"), "-o", str(tmp_path / "x.json")],
                       capture_output=True, text=True)
    assert r.returncode == 2 and "fingerprint" in r.stderr
