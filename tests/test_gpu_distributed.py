"""The distributed hot path on the GPU (quantc/distributed.hpp, comm.hpp).

* NCCL communicator (world 1 — one GPU per box here): the distributed
  collect_stats and the sample- / candidate-sharded searches run through
  ncclAllReduce / ncclAllGather and equal the single-process reference.
* World 2 over gloo with both ranks on cuda:0 (their kernels never wait on
  each other; only the host collectives synchronise them): calibration images
  sharded, candidate batches sharded, calibration samples sharded — every
  rank's statistics, thresholds and SearchResult equal the reference's
  single-process collect_stats and serial search on the whole set."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_14949_b200 import fixtures as F
from paper_2103_14949_b200 import quantc as Q

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_IMG = 10
SEARCHES = [("greedy", dict(rounds=2, tol=0.05)), ("random", dict(n=10, seed=3)),
            ("anneal", dict(steps=10, t0=0.05, decay=0.9, seed=4))]


def _model():
    return F.small_cnn(channels=8, image=16)


def _graphs(q, m):
    g = q.graph(m.doc, m.blob)
    spec = q.parse_spec(F.spec_fixture("int8_int32"))
    topo = q.generate_topology(g, spec)
    sim = q.insert_simulated_quantize(g, topo)
    return g, spec, topo, sim


def _stats_tuple(st):
    return {k: (v["min"], v["max"], v["absmax"], v["sample_count"], v["counts"].tolist())
            for k, v in st.per_edge().items()}


def _reference(ref):
    """Single-process reference: stats, thresholds, serial searches."""
    m = _model()
    data = m.data(N_IMG)
    g, spec, topo, sim = _graphs(ref, m)
    ds = ref.dataset(data)
    st = ref.collect_stats(g, ds, 2048, ref.simulated_edge_indices(g, topo))
    thr = st.estimate_thresholds("quantile", quantile=0.99, pow2=True)
    ev = ref.evaluator(sim, spec, topo, thr, st, ds)
    res = {}
    for method, kw in SEARCHES:
        r = ref.search(method, ev.space(), evaluator=ev, **kw)
        res[method] = (r.best, r.best_loss, r.evaluations, repr(r.trace))
    return _stats_tuple(st), thr, res


def test_nccl_world1_equals_reference(b200, ref):
    comm = b200.comm_nccl(0, 1, b200.nccl_unique_id())
    m = _model()
    data = m.data(N_IMG)
    g, spec, topo, sim = _graphs(b200, m)
    ds = b200.dataset(data)
    st = b200.collect_stats_dist(g, ds, comm, 2048, b200.simulated_edge_indices(g, topo))
    rst, rthr, rres = _reference(ref)
    assert _stats_tuple(st) == rst
    thr = st.estimate_thresholds("quantile", quantile=0.99, pow2=True)
    assert thr == rthr
    ev = b200.evaluator(sim, spec, topo, thr, st, ds)
    for mode in ("samples", "candidates", "local"):
        for method, kw in SEARCHES:
            r = b200.search_batched(method, ev.space(), evaluator=ev, comm=comm, mode=mode,
                                    width=4, **kw)
            assert (r.best, r.best_loss, r.evaluations, repr(r.trace)) == rres[method], \
                (mode, method)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["QUANTC_DEVICE"] = "0"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q = Q.load_b200()
        comm = q.comm_torch()
        m = _model()
        data = m.data(N_IMG)
        lo, hi = [(0, 6), (6, 10)][rank]  # uneven shards
        g, spec, topo, sim = _graphs(q, m)
        shard = q.dataset(np.ascontiguousarray(data[lo:hi]))
        st = q.collect_stats_dist(g, shard, comm, 2048, q.simulated_edge_indices(g, topo))
        thr = st.estimate_thresholds("quantile", quantile=0.99, pow2=True)
        out = {"stats": _stats_tuple(st), "thr": thr}
        # candidates sharded: every rank holds the full calibration set
        full = q.dataset(data)
        ev_full = q.evaluator(sim, spec, topo, thr, st, full)
        # samples sharded: the evaluator holds this rank's shard
        ev_shard = q.evaluator(sim, spec, topo, thr, st, shard)
        for method, kw in SEARCHES:
            r = q.search_batched(method, ev_full.space(), evaluator=ev_full, comm=comm,
                                 mode="candidates", width=4 * world, **kw)
            out[("candidates", method)] = (r.best, r.best_loss, r.evaluations, repr(r.trace))
            r = q.search_batched(method, ev_shard.space(), evaluator=ev_shard, comm=comm,
                                 mode="samples", width=4, **kw)
            out[("samples", method)] = (r.best, r.best_loss, r.evaluations, repr(r.trace))
        out_q.put((rank, out, None))
    except BaseException as e:  # pragma: no cover
        import traceback
        out_q.put((rank, None, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_sharded_equals_reference(ref):
    rst, rthr, rres = _reference(ref)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, res, err = q.get(timeout=600)
        assert err is None, err
        got[rank] = res
    for p in procs:
        p.join(timeout=60)
    for rank in range(world):
        o = got[rank]
        assert o["stats"] == rst
        assert o["thr"] == rthr
        for method, _ in SEARCHES:
            assert o[("candidates", method)] == rres[method], (rank, method)
            assert o[("samples", method)] == rres[method], (rank, method)
