"""N>1 path on CPU: world_size-2 gloo runs of paper_2103_14949_b200/parallel.py.
The per-rank compute is the reference oracle (CPU); what is under test is the
product's sharding + exact all-reduce merge logic, which must reproduce the
single-process reference collect_stats and losses bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_14949_b200 import fixtures as F
from paper_2103_14949_b200 import parallel as P
from paper_2103_14949_b200 import quantc as Q

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "oracle", "_ref", "libquantc_ref.so")
PORT = os.path.join(REPO, "oracle", "_build", "libqcoracle.so")


def test_shard_range_partitions():
    for n in (0, 1, 7, 16, 1024, 1001):
        for w in (1, 2, 3, 4, 8):
            spans = [P.shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests import oracle_port
        ref = Q.Quantc(REF)
        orc = oracle_port.load(PORT)
        m = F.small_cnn(channels=8, image=16)
        data = m.data(10)
        g = ref.graph(m.doc, m.blob)
        spec = ref.parse_spec(F.spec_fixture("int8_int32"))
        topo = ref.generate_topology(g, spec)
        edges = ref.simulated_edge_indices(g, topo)
        src = [g.edge_order()[k][0] for k in edges]
        lo_i, hi_i = P.shard_range(len(data), rank, world)
        shard = data[lo_i:hi_i]

        def activations(x):
            # producer tensors of the target edges for one sample (reference fp32)
            return {nid: ref.eval_fp32_values(g, x, [nid]) for nid in sorted(set(src))}

        acts = [activations(x) for x in shard]

        def local_extrema(es):
            lo = np.full(len(es), np.inf)
            hi = np.full(len(es), -np.inf)
            for a in acts:
                for i, k in enumerate(es):
                    v = a[src[edges.index(k)]].astype(np.float64)
                    lo[i] = min(lo[i], v.min())
                    hi[i] = max(hi[i], v.max())
            return lo, hi

        def local_hist(es, absmax, bins):
            out = np.zeros((len(es), bins), np.int64)
            for a in acts:
                for i, k in enumerate(es):
                    out[i] += orc.histogram(a[src[edges.index(k)]], float(absmax[i]), bins)
            return out.reshape(-1)

        stats = P.sharded_collect_stats(edges, len(data), 2048, local_extrema, local_hist)

        # sharded search losses: per-rank agreement counts over the local shard
        full = ref.dataset(data)
        st_full = ref.collect_stats(g, full, 2048, edges)
        thr = st_full.estimate_thresholds("quantile", pow2=False)
        sim = ref.insert_simulated_quantize(g, topo)
        ev = ref.evaluator(sim, spec, topo, thr, st_full, full)
        refs = ev.reference_predictions()
        shard_ds = ref.dataset(shard)

        def local_counts(cands):
            out = []
            for c in cands:
                p = ref.predict_top1(sim, shard_ds, 1, ev.bind(c))
                out.append(int((p == refs[lo_i:hi_i]).sum()))
            return np.array(out, np.int64)

        sev = P.ShardedEvaluator(local_counts, len(data))
        sp = ev.space()
        cands = [sp.all_hi(), sp.all_lo(), [6] * len(sp.hi)]
        sharded_losses = sev.losses(cands)
        if rank == 0:
            expect = {k: st_full.get(k) for k in edges}
            out_q.put(("ok", {k: (v["min"], v["max"], v["absmax"], v["counts"].tolist())
                              for k, v in stats.items()},
                       {k: (v["min"], v["max"], v["absmax"], v["counts"].tolist())
                        for k, v in expect.items()},
                       sharded_losses.tolist(), ev.losses(cands).tolist()))
    except Exception as e:  # surface to the parent
        import traceback
        out_q.put(("err", traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not (os.path.exists(REF) and os.path.exists(PORT)), reason="oracle not built")
def test_sharded_calibration_and_losses_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
    assert res[0] == "ok", res[1]
    _, got, want, sl, fl = res
    assert got == want
    assert sl == fl
