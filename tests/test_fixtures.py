"""quantc::fixtures (include/quantc/fixtures.hpp; reference fixtures.hpp:13-60,
declared only; contract SPEC.md:734-782).  CPU: the C++ header compiles and
behaves as declared (tests/cpp/fixtures_check.cpp, built against the
library), and the committed fixture files (tests/fixtures/quantc, written by
write_all) regenerate byte for byte (verify_committed)."""
import os
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COMMITTED = os.path.join(REPO, "tests", "fixtures", "quantc")


def test_fixtures_cpp_api(tmp_path):
    pkg = os.path.join(REPO, "paper_2103_14949_b200")
    vendor = os.path.join(pkg, "csrc", "build", "vendor")
    exe = tmp_path / "fixtures_check"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{REPO}/include", f"-I{vendor}",
                    os.path.join(REPO, "tests", "cpp", "fixtures_check.cpp"),
                    f"-L{pkg}", "-lquantc_b200", f"-Wl,-rpath,{pkg}", "-o", str(exe)],
                   check=True, capture_output=True)
    r = subprocess.run([str(exe), str(tmp_path / "scratch"), COMMITTED], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    assert "ok" in r.stdout


def test_committed_fixtures_regenerate(b200):
    b200.fixtures_verify_committed(COMMITTED)
    g = b200.load_graph(os.path.join(COMMITTED, "small_cnn.json"))
    assert g.validate() == []
    assert b200.load_dataset(os.path.join(COMMITTED, "small_cnn_evaluation.json")).n == 256
