"""SPEC acceptance 4 on the CPU: the committed (or a freshly written) small_cnn
fixture run through the reference library (oracle/_ref: stats, thresholds,
evaluator, greedy, eval_int) with this repo's host-only realize().  Used to
tune the fixture generator without a GPU; the -m gpu test runs the same
pipeline on the B200 library."""
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

fx = sys.argv[1] if len(sys.argv) > 1 else os.path.join(REPO, "tests", "fixtures", "quantc")
b = Q.load_b200()
ref = Q.load(os.path.join(REPO, "oracle", "_ref", "libquantc_ref.so"))


def samples(name):
    man = json.load(open(os.path.join(fx, name + ".json")))
    out = []
    for s in man:
        r = s["inputs"][0]
        n = int(np.prod(r["shape"]))
        blob = open(os.path.join(fx, r["file"]), "rb").read()
        out.append(np.frombuffer(blob, np.float32, n, r["offset"]).reshape(r["shape"]))
    return np.stack(out)


g_b = b.load_graph(os.path.join(fx, "small_cnn.json"))
g = g_b.copy_to(ref)
spec_txt = open(os.path.join(fx, "specs", "int8_int32.json")).read()
spec = ref.parse_spec(spec_txt)
topo = ref.generate_topology(g, spec)
sim = ref.insert_simulated_quantize(g, topo)
cal, evx = samples("small_cnn_calibration"), samples("small_cnn_evaluation")
ds = ref.dataset(cal)
st = ref.collect_stats(g, ds, 2048, ref.simulated_edge_indices(g, topo))
fp32 = ref.predict_top1(g, ref.dataset(evx))
for method in sys.argv[2:] or ["max"]:
    thr = st.estimate_thresholds(method)
    ev = ref.evaluator(sim, spec, topo, thr, st, ds)
    for tol in (0.0, 0.01):
        res = ref.search("greedy", ev.space(), evaluator=ev, rounds=1, tol=tol)
        strat = ev.strategy_for(res.best)
        sim_b = b.insert_simulated_quantize(g_b, b.generate_topology(g_b, b.parse_spec(spec_txt)))
        R = b.realize(sim_b, strat, b.parse_spec(spec_txt)).copy_to(ref)
        got = [int(np.argmax(np.asarray(ref.eval_int(R, x, trap=True)[0], np.float64).reshape(-1)))
               for x in evx]
        print(method, "tol", tol, "bits", list(res.best), "cal loss", res.best_loss,
              "eval agree", float(np.mean(np.asarray(got) == fp32)), flush=True)
