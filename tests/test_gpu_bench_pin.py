"""The benchmarked configuration, pinned to the reference.

bench.py times ResNet-50 at 224x224 with 1000 classes, quantile-0.999 pow2
thresholds on the int8_int32 spec, candidates evaluated four at a time
through grouped tcgen05 launches.  Here that exact pipeline runs on 8 of the
bench's images (seed 9) and is compared with the reference implementation
(oracle/_ref, the reference sources compiled here) on the same inputs:

  * statistics -> thresholds: identical (reference collect_stats, calibration.cpp:37-115);
  * the fp32 reference predictions: identical (search.cpp:313);
  * bindings of every candidate: identical QParams (search.cpp:316-401);
  * fp32 score rows of every candidate and image, BYTE for byte, against the
    reference's eval_fp32 under the same binding (interpreter.cpp:487-492),
    through BOTH the grouped (G = 4) and the one-candidate path;
  * losses and per-image predictions (search.cpp:421-428, interpreter.cpp:533-556).

Candidates: all_hi, all_lo, two random, and four of bench.py's single-slot
probes.  The reference side runs (candidate, image) forwards on all host
cores (ctypes releases the GIL)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import bench
from paper_2103_14949_b200 import fixtures as F

pytestmark = pytest.mark.gpu

N_IMG = 8


def _pipeline(q, model, data):
    g = q.graph(model.doc, model.blob)
    spec = q.parse_spec(F.spec_fixture("int8_int32"))
    topo = q.generate_topology(g, spec)
    sim = q.insert_simulated_quantize(g, topo)
    ds = q.dataset(data)
    st = q.collect_stats(g, ds, 2048, q.simulated_edge_indices(g, topo))
    thr = st.estimate_thresholds("quantile", quantile=0.999, pow2=True)
    return dict(g=g, spec=spec, topo=topo, sim=sim, ds=ds, st=st, thr=thr)


@pytest.fixture(scope="module")
def pinned(b200, ref):
    model = F.resnet(50)
    data = model.data(64, seed=9)[:N_IMG]  # the bench's first images
    a = _pipeline(b200, model, data)
    r = _pipeline(ref, model, data)
    a["ev"] = b200.evaluator(a["sim"], a["spec"], a["topo"], a["thr"], a["st"], a["ds"])
    r["ev"] = ref.evaluator(r["sim"], r["spec"], r["topo"], r["thr"], r["st"], r["ds"])
    sp = a["ev"].space()
    rng = np.random.default_rng(3)
    cands = ([sp.all_hi(), sp.all_lo()]
             + [[int(rng.integers(lo, hi + 1)) for lo, hi in zip(sp.lo, sp.hi)] for _ in range(2)]
             + bench.candidates(sp, 4))
    # the reference's fp32 scores of every (candidate, image)
    bindings = [a["ev"].bind(c) for c in cands]
    jobs = [(ci, i) for ci in range(len(cands)) for i in range(N_IMG)]

    def one(job):
        ci, i = job
        return ref.eval_fp32(r["sim"], data[i], bindings[ci])

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 8) as ex:
        outs = list(ex.map(one, jobs))
    ref_scores = np.stack(outs).reshape(len(cands), N_IMG, -1).astype(np.float32)
    return dict(a=a, r=r, model=model, data=data, cands=cands, ref_scores=ref_scores)


def test_collect_stats_bit_exact_at_224(pinned):
    """collect_stats over the 8 bench images at 224x224 (all 191 simulated
    edges): min / max / absmax / sample_count and all 2048 int64 counts equal
    the reference's (calibration.cpp:37-115)."""
    a, r = pinned["a"], pinned["r"]
    assert a["st"].edges() == r["st"].edges()
    assert len(r["st"].edges()) == 191
    for k in r["st"].edges():
        ea, er = a["st"].get(k), r["st"].get(k)
        assert (ea["min"], ea["max"], ea["absmax"], ea["sample_count"]) == \
            (er["min"], er["max"], er["absmax"], er["sample_count"]), k
        np.testing.assert_array_equal(ea["counts"], er["counts"], err_msg=f"edge {k}")


def test_thresholds_and_refs_identical(pinned):
    a, r = pinned["a"], pinned["r"]
    assert a["thr"] == r["thr"]
    np.testing.assert_array_equal(a["ev"].reference_predictions(),
                                  r["ev"].reference_predictions())
    assert a["ev"].space() == r["ev"].space()


def test_bindings_identical(pinned):
    a, r = pinned["a"], pinned["r"]
    for c in pinned["cands"]:
        ba, br = a["ev"].bind(c), r["ev"].bind(c)
        assert ba.keys() == br.keys()
        for k, p in br.items():
            assert ba[k].as_dict() == p.as_dict(), k


@pytest.mark.parametrize("group", [4, 1])
def test_scores_bytes_equal_reference(pinned, cuda_lib, group):
    """Grouped (G = 4, the bench's path) and single-candidate score rows
    equal the reference's eval_fp32 bytes for every candidate and image."""
    a = pinned["a"]
    f0 = cuda_lib.counters()["fused_batches"]
    got = a["ev"].scores(pinned["cands"], group=group)
    assert cuda_lib.counters()["fused_batches"] - f0 >= len(pinned["cands"]), \
        "the fused tcgen05 engine was not used"
    exp = pinned["ref_scores"]
    assert got.shape == exp.shape
    bad = got.view(np.uint32) != exp.view(np.uint32)
    assert not bad.any(), (int(bad.sum()), np.argwhere(bad)[:5].tolist())


def test_losses_and_predictions_equal_reference(pinned, b200):
    a, r = pinned["a"], pinned["r"]
    cands = pinned["cands"]
    refs = r["ev"].reference_predictions()
    ref_preds = pinned["ref_scores"].argmax(axis=2)  # first maximum, like argmax_class
    ref_losses = 1.0 - (ref_preds == refs[None, :]).sum(axis=1) / float(N_IMG)
    np.testing.assert_array_equal(a["ev"].losses(cands), ref_losses)
    for ci, c in enumerate(cands[:3]):
        np.testing.assert_array_equal(
            b200.predict_top1(a["sim"], a["ds"], 0, a["ev"].bind(c)), ref_preds[ci])
