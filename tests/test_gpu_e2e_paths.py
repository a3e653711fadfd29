"""predict_top1 through the C-ABI with the dataset page-locked (default: DMA
straight from the samples) and not (QUANTC_PIN_MAX_MB=0: packed through the
pinned staging buffers) gives identical predictions (reference equality of
predict_top1 is covered by test_gpu_parity.py)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2103_14949_b200 import fixtures as F

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, {repo!r})
from paper_2103_14949_b200 import fixtures as F, quantc as Q
b = Q.load_b200()
m = F.resnet(18, image=64, classes=10, width=16)
g = b.graph(m.doc, m.blob)
spec = b.parse_spec(F.spec_fixture("int8_int32"))
topo = b.generate_topology(g, spec)
sim = b.insert_simulated_quantize(g, topo)
data = m.data(24)
ds = b.dataset(data)
st = b.collect_stats(g, ds, 2048, b.simulated_edge_indices(g, topo))
thr = st.estimate_thresholds("quantile", quantile=0.999, pow2=True)
ev = b.evaluator(sim, spec, topo, thr, st, ds)
print(json.dumps(b.predict_top1(sim, ds, 0, ev.bind(ev.space().all_hi())).tolist()))
"""


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(repo=REPO)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_pinned_and_staged_uploads_agree():
    pinned = _run({})
    staged = _run({"QUANTC_PIN_MAX_MB": "0"})
    assert pinned == staged
    assert len(pinned) == 24
