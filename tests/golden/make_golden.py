"""Generates tests/golden/*.json from the REFERENCE implementation compiled
in this container (oracle/_ref/libquantc_ref.so, built from
/root/reference/proj/src by oracle/Makefile).  Committed so the known answers
travel without /root/reference.  Run:  python tests/golden/make_golden.py"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
from paper_2103_14949_b200 import fixtures as F  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402


def main():
    ref = Q.load(os.path.join(REPO, "oracle", "_ref", "libquantc_ref.so"))
    out = {}
    # SPEC.md simulate examples (verified against the compiled reference)
    out["compute_scale"] = [[t, b, s, ref.compute_scale(t, b, s)]
                            for t, b, s in [(1.0, 8, 1), (6.0, 6, 1), (1.0, 8, 0), (0.37, 5, 1)]]
    out["quant_bounds"] = [[b, s, *ref.quant_bounds(b, s)] for b, s in [(8, 1), (6, 1), (8, 0), (16, 1)]]
    sqv = []
    for x, t, b in [(0.5, 1.0, 8), (2.0, 1.0, 8), (0.004, 1.0, 8), (-0.77, 0.9, 5), (1e-3, 1e-8, 8)]:
        sqv.append([x, t, b, ref.simulated_quantize_value(x, Q.QParams.symmetric(t, b))])
    out["sim_quant_value"] = sqv
    rng = np.random.default_rng(123)
    tuples = []
    for _ in range(200):
        t = float(np.exp(rng.uniform(-6, 6)))
        bit = int(rng.integers(2, 9))
        sign = int(rng.integers(0, 2))
        zp = 0 if sign else int(rng.integers(0, 1 << bit))
        acc = int(rng.integers(0, 2))
        x = float(np.float32(rng.standard_normal() * t * 1.5))
        p = Q.QParams.make(t, bit, sign, Q.I8 if sign else Q.U8, zero_point=zp,
                           acc_dtype=Q.I16 if acc else Q.NONE, acc_scale=t / 300 if acc else 0.0)
        tuples.append([x, t, bit, sign, zp, acc, t / 300 if acc else 0.0,
                       ref.simulated_quantize_value(x, p)])
    out["sim_quant_tuples"] = tuples
    out["round_pow2"] = [[v, ref.round_pow2(v)] for v in (3.2, 2.0, 1.5, 0.3, 1e-8, 7.99)]
    out["asymmetric_zero_point"] = [[mn, t, b, ref.asymmetric_zero_point(mn, t, b)]
                                    for mn, t, b in [(-1.0, 4.0, 8), (0.5, 2.0, 4), (-10.0, 3.0, 8)]]
    # quantile: values 1..100 into B=100 bins over [0,100]
    counts = np.ones(100, np.int64)
    out["quantile_1_100"] = ref.threshold_quantile(counts, 100.0, 0.99)
    kl = []
    for seed in range(50):
        r = np.random.default_rng(seed)
        bins = int(r.choice([16, 32, 64, 128, 256]))
        tb = int(r.integers(1, int(np.log2(bins)) + 1))
        h = r.integers(0, 50, bins) * (r.random(bins) < 0.7)
        h[0] += 1
        kl.append([h.tolist(), 3.5, tb, ref.threshold_kl(h, 3.5, tb)])
    out["kl_random"] = kl
    h0 = np.zeros(2048, np.int64)
    h0[0] = 1000
    out["kl_all_mass_bin0"] = ref.threshold_kl(h0, 5.0, 8)
    # small CNN pipeline (BASELINE config 0)
    m = F.small_cnn()
    data = m.data(16)
    g = ref.graph(m.doc, m.blob)
    spec = ref.parse_spec(F.spec_fixture("int8_int32"))
    topo = ref.generate_topology(g, spec)
    sim = ref.insert_simulated_quantize(g, topo)
    ds = ref.dataset(data)
    edges = ref.simulated_edge_indices(g, topo)
    st = ref.collect_stats(g, ds, 2048, edges)
    pipe = {"edges": edges, "stats": {}, "thresholds": {}}
    for k in edges:
        e = st.get(k)
        pipe["stats"][str(k)] = {"min": e["min"], "max": e["max"], "absmax": e["absmax"],
                                 "counts_nonzero": {str(i): int(c) for i, c in
                                                    enumerate(e["counts"]) if c}}
    for meth, pw in [("max", False), ("quantile", False), ("kl", False), ("quantile", True)]:
        pipe["thresholds"][f"{meth}{'_pow2' if pw else ''}"] = {
            str(k): v for k, v in st.estimate_thresholds(meth, pow2=pw).items()}
    thr = st.estimate_thresholds("quantile", pow2=False)
    ev = ref.evaluator(sim, spec, topo, thr, st, ds)
    sp = ev.space()
    pipe["refs"] = ev.reference_predictions().tolist()
    cands = [sp.all_hi(), sp.all_lo(), [6] * len(sp.hi), [8, 4, 8, 4, 8, 4, 8, 4]]
    pipe["candidates"] = cands
    pipe["losses"] = ev.losses(cands).tolist()
    res = ref.search("greedy", sp, evaluator=ev, rounds=1, tol=0.05)
    pipe["greedy"] = {"best": res.best, "best_loss": res.best_loss,
                      "evaluations": res.evaluations}
    out["small_cnn_pipeline"] = pipe
    json.dump(out, open(os.path.join(HERE, "reference_golden.json"), "w"), indent=1)
    print("wrote", os.path.join(HERE, "reference_golden.json"))


if __name__ == "__main__":
    main()
