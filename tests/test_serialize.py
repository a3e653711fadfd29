"""serialize.hpp files (reference proj/include/quantc/serialize.hpp:18-56,
formats SPEC.md:102 graph file, :382 stats file): save -> load round trips
through the B200 library's C-ABI, checked against the reference build's own
evaluation of the same graph.  Host code only; runs on CPU."""
import json

import numpy as np
import pytest

from paper_2103_14949_b200 import fixtures as F


def _fnv(data: bytes, seed=1469598103934665603):
    h = seed
    for b in data:
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def test_fnv1a64_known_answers(b200):
    # published FNV-1a 64 test vectors under the published offset basis
    basis = 0xCBF29CE484222325
    assert b200.fnv1a64(b"", seed=basis) == basis
    assert b200.fnv1a64(b"a", seed=basis) == 0xAF63DC4C8601EC8C
    assert b200.fnv1a64(b"foobar", seed=basis) == 0x85944171F73967E8
    # the default seed is the reference's declared one (serialize.hpp:53,
    # 1469598103934665603 -- the basis without its last digit), kept as is
    assert b200.fnv1a64(b"") == 1469598103934665603
    assert b200.fnv1a64(b"foobar") == _fnv(b"foobar", 1469598103934665603)
    blob = np.random.default_rng(0).bytes(999)
    assert b200.fnv1a64(blob, seed=12345) == _fnv(blob, 12345)


def test_graph_file_round_trip(b200, ref, tmp_path):
    model = F.small_cnn()
    g = b200.graph(model.doc, model.blob)
    path = tmp_path / "model.json"
    g.save(path)
    assert (tmp_path / "model.bin").exists()
    doc = json.loads(path.read_text())
    # SPEC.md graph module: the sidecar ref lives in the constant's attrs
    refs = [n["attrs"]["payload"] for n in doc["nodes"] if "payload" in n.get("attrs", {})]
    assert refs and all(set(r) == {"file", "offset", "dtype", "shape"} for r in refs)
    assert all(r["file"] == "model.bin" for r in refs)
    g2 = b200.load_graph(path)
    assert g2.to_json() == g.to_json()
    assert g2.blob() == g.blob()
    assert g2.fingerprint() == g.fingerprint()
    # the loaded graph evaluates like the original on the reference interpreter
    x = model.data(1)[0]
    np.testing.assert_array_equal(ref.eval_fp32(g2.copy_to(ref), x),
                                  ref.eval_fp32(g.copy_to(ref), x))


def test_graph_fingerprint_sensitive_to_payload(b200):
    model = F.small_cnn()
    g = b200.graph(model.doc, model.blob)
    blob = bytearray(model.blob)
    blob[0] ^= 1
    g2 = b200.graph(model.doc, bytes(blob))
    assert g.fingerprint() != g2.fingerprint()


def test_realized_graph_file_round_trip(b200, ref, tmp_path):
    """Integer payloads (int8 weights, int32 biases) keep their natural width
    in the sidecar and reload bit-exact."""
    doc, blob = F.int_conv_probe(requant=(1 << 30, 41, 7, -3))
    g = b200.graph(doc, blob)
    g.save(tmp_path / "int.json")
    d = json.loads((tmp_path / "int.json").read_text())
    dts = {n["attrs"]["payload"]["dtype"] for n in d["nodes"] if "payload" in n["attrs"]}
    assert dts & {"int8", "int32"}, dts
    g2 = b200.load_graph(tmp_path / "int.json")
    assert g2.to_json() == g.to_json() and g2.blob() == g.blob()
    x = np.random.default_rng(1).normal(0, 2, (2, 16, 12, 12)).astype(np.float32)
    y1, t1 = ref.eval_int(g.copy_to(ref), x)
    y2, t2 = ref.eval_int(g2.copy_to(ref), x)
    assert t1 == t2
    np.testing.assert_array_equal(y1, y2)


def test_stats_file_round_trip(b200, ref, tmp_path):
    model = F.small_cnn()
    g = ref.graph(model.doc, model.blob)
    spec = ref.parse_spec(F.spec_fixture("int8_int32"))
    topo = ref.generate_topology(g, spec)
    st = ref.collect_stats(g, ref.dataset(model.data(4)), 512,
                           ref.simulated_edge_indices(g, topo))
    mine = b200.make_stats(st.per_edge())
    mine.save(tmp_path / "stats.json")
    doc = json.loads((tmp_path / "stats.json").read_text())
    e0 = doc["per_edge"][str(st.edges()[0])]
    assert set(e0) == {"min", "max", "absmax", "bins", "counts", "samples"}
    assert e0["bins"] == 512
    back = b200.load_stats(tmp_path / "stats.json")
    assert back.edges() == st.edges()
    for k in st.edges():
        a, b = st.get(k), back.get(k)
        assert (a["min"], a["max"], a["absmax"], a["sample_count"]) == (
            b["min"], b["max"], b["absmax"], b["sample_count"])
        np.testing.assert_array_equal(a["counts"], b["counts"])
    # (the B200 library sweeps thresholds on the device: evaluate the reloaded
    # file through the reference build instead)
    again = ref.make_stats(back.per_edge())
    for method in ("max", "quantile", "kl"):
        assert again.estimate_thresholds(method, quantile=0.999) == \
            st.estimate_thresholds(method, quantile=0.999)


def test_load_errors_are_io_errors(b200, tmp_path):
    import pytest
    from paper_2103_14949_b200 import quantc as Q
    with pytest.raises(Q.QuantcError):
        b200.load_graph(tmp_path / "missing.json")
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(Q.QuantcError):
        b200.load_stats(tmp_path / "bad.json")
    model = F.small_cnn()
    b200.graph(model.doc, model.blob).save(tmp_path / "m.json")
    (tmp_path / "m.bin").write_bytes(b"\0" * 8)  # truncated sidecar
    with pytest.raises(Q.QuantcError):
        b200.load_graph(tmp_path / "m.json")


def test_cpp_dataset_strategy_trace_round_trip(tmp_path):
    """The C++-only files (dataset manifest, strategy, trace): a small program
    built against include/quantc/serialize.hpp and the B200 library."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_2103_14949_b200")
    vendor = os.path.join(pkg, "csrc", "build", "vendor")
    exe = tmp_path / "roundtrip"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{root}/include", f"-I{vendor}",
                    os.path.join(root, "tests", "cpp", "serialize_roundtrip.cpp"),
                    f"-L{pkg}", "-lquantc_b200", f"-Wl,-rpath,{pkg}", "-o", str(exe)],
                   check=True, capture_output=True)
    r = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "ok" in r.stdout


def test_graph_file_spec_forms_load(b200, tmp_path):
    """A graph file written to SPEC.md by another tool loads: the ref as
    attrs.payload, the ref keys directly in attrs, or (round-1 files) a
    node-level payload — all give the same graph."""
    model = F.small_cnn()
    g = b200.graph(model.doc, model.blob)
    g.save(tmp_path / "m.json")
    doc = json.loads((tmp_path / "m.json").read_text())
    flat = json.loads(json.dumps(doc))
    legacy = json.loads(json.dumps(doc))
    for a, b in zip(flat["nodes"], legacy["nodes"]):
        if "payload" in a.get("attrs", {}):
            ref = a["attrs"].pop("payload")
            a["attrs"].update(ref)
            b["payload"] = b["attrs"].pop("payload")
    for name, d in (("flat", flat), ("legacy", legacy)):
        (tmp_path / f"{name}.json").write_text(json.dumps(d))
        (tmp_path / f"{name}.bin").write_bytes((tmp_path / "m.bin").read_bytes())
        for n in d["nodes"]:
            for r in ([n["attrs"]] if "file" in n.get("attrs", {}) else []) + \
                     ([n["payload"]] if "payload" in n else []):
                r["file"] = f"{name}.bin"
        (tmp_path / f"{name}.json").write_text(json.dumps(d))
        g2 = b200.load_graph(tmp_path / f"{name}.json")
        assert g2.to_json() == g.to_json(), name
        assert g2.blob() == g.blob(), name


def test_malformed_files_raise_io_error(b200, tmp_path):
    from paper_2103_14949_b200 import quantc as Q
    bad_stats = tmp_path / "s.json"
    bad_stats.write_text('{"per_edge": {"x": {"min": 0, "max": 1, "absmax": 1, '
                         '"counts": [1], "samples": 1}}}')
    with pytest.raises(Q.QuantcError) as e:
        b200.load_stats(bad_stats)
    assert "malformed stats" in str(e.value)
    bad_stats.write_text('[1, 2]')
    with pytest.raises(Q.QuantcError):
        b200.load_stats(bad_stats)
