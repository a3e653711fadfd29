"""The sharded calibration passes on the GPU (parallel.B200Local over the
C-ABI qc_collect_extrema / qc_collect_histograms, merged exactly as the NCCL
path merges them) equal the reference's collect_stats on the whole set —
with the pass-1 -> pass-2 activation handoff and without it."""
import numpy as np
import pytest

from paper_2103_14949_b200 import fixtures as F
from paper_2103_14949_b200 import parallel as P

pytestmark = pytest.mark.gpu


def _edges(q, m):
    g = q.graph(m.doc, m.blob)
    spec = q.parse_spec(F.spec_fixture("int8_int32"))
    return g, q.simulated_edge_indices(g, q.generate_topology(g, spec))


@pytest.mark.parametrize("handoff", [True, False])
def test_sharded_passes_equal_reference_collect_stats(b200, ref, handoff):
    m = F.resnet(18, image=32, classes=10, width=8)
    data = m.data(10)
    gr, edges = _edges(ref, m)
    want = ref.collect_stats(gr, ref.dataset(data), 2048, edges)
    g, edges_b = _edges(b200, m)
    assert edges_b == edges
    shards = [b200.dataset(data[a:b]) for a, b in (P.shard_range(10, r, 3) for r in range(3))]
    locs = [P.B200Local(b200, g, s) for s in shards]
    ext = [loc.extrema(edges) for loc in locs]
    lo = np.min([e[0] for e in ext], axis=0)
    hi = np.max([e[1] for e in ext], axis=0)
    absmax = np.maximum(np.abs(lo), np.abs(hi))
    if not handoff:
        # a pass 1 on another shard supersedes the handoff: every shard's
        # pass 2 recomputes its forward
        locs[0].extrema(edges[:3])
    counts = sum(loc.histograms(edges, absmax, 2048) for loc in locs)
    counts = counts.reshape(len(edges), 2048)
    for i, k in enumerate(edges):
        w = want.get(k)
        assert (lo[i], hi[i], absmax[i]) == (w["min"], w["max"], w["absmax"]), k
        np.testing.assert_array_equal(counts[i], w["counts"], err_msg=f"edge {k}")


def test_histogram_handoff_used_for_last_shard(b200):
    # the shard whose pass 1 ran last hands its activations to pass 2:
    # identical counts either way
    m = F.small_cnn()
    data = m.data(6)
    g, edges = _edges(b200, m)
    loc = P.B200Local(b200, g, b200.dataset(data))
    lo, hi = loc.extrema(edges)
    absmax = np.maximum(np.abs(lo), np.abs(hi))
    with_handoff = loc.histograms(edges, absmax, 2048)
    without = loc.histograms(edges, absmax, 2048)  # handoff consumed: recompute
    np.testing.assert_array_equal(with_handoff, without)
