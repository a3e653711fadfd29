"""quantc CLI: exit codes without a GPU — 1 usage, 2 validation
(unreadable / malformed inputs name the path)."""
import os
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(REPO, "paper_2103_14949_b200", "quantc")
FX = os.path.join(REPO, "tests", "fixtures", "quantc")


def _run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True)


def test_usage_errors_exit_1():
    assert _run().returncode == 1
    assert _run("frobnicate").returncode == 1
    assert _run("calibrate", "-m").returncode == 1
    r = _run("calibrate", "-m", os.path.join(FX, "small_cnn.json"))
    assert r.returncode == 1 and "missing" in r.stderr


def test_missing_or_bad_files_exit_2(tmp_path):
    missing = str(tmp_path / "nope.json")
    r = _run("calibrate", "-m", os.path.join(FX, "small_cnn.json"), "-s", missing,
             "-d", os.path.join(FX, "small_cnn_calibration.json"), "-o", str(tmp_path / "s.json"))
    assert r.returncode == 2 and "nope.json" in r.stderr
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    r = _run("calibrate", "-m", str(bad), "-s", os.path.join(FX, "specs", "int8_int32.json"),
             "-d", os.path.join(FX, "small_cnn_calibration.json"), "-o", str(tmp_path / "s.json"))
    assert r.returncode == 2 and "bad.json" in r.stderr
