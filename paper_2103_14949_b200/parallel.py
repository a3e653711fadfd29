"""Multi-GPU driver: one process per GPU, calibration and candidate evaluation
sharded over ranks, exact NCCL all-reduce merges.

The reference's only parallelism is a thread pool over samples whose per-
sample partials merge associatively (calibration.cpp:62-113, interpreter.cpp:
546).  Here the unit is a rank: rank r owns the contiguous sample range
shard_range(N, r, world); the merges are

  * extrema  : all_reduce(MIN / MAX) of float64 per edge, between the passes
  * histogram: all_reduce(SUM) of int64 [edges, bins] against the global absmax
  * search   : all_reduce(SUM) of int64 agreement counts per candidate batch

All three are exact (min/max and integer sums are order-free), so results are
bit-identical to one GPU and to the reference.  The per-rank compute is
injectable (`local_*` callables) so the merge logic runs under gloo on CPU in
tests; `B200Local` wires it to the B200 library's C-ABI.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

from . import quantc as Q


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced partition of n samples (first n % world ranks get one more)."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def _device(group) -> torch.device:
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _single() -> bool:
    return not (dist.is_available() and dist.is_initialized())


def allreduce_extrema(mins: Sequence[float], maxs: Sequence[float], group=None):
    if _single():  # one process: the local extrema are the global ones
        return np.asarray(mins, np.float64), np.asarray(maxs, np.float64)
    dev = _device(group)
    lo = torch.tensor(list(mins), dtype=torch.float64, device=dev)
    hi = torch.tensor(list(maxs), dtype=torch.float64, device=dev)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    return lo.cpu().numpy(), hi.cpu().numpy()


def allreduce_counts(counts: np.ndarray, group=None) -> np.ndarray:
    if _single():
        return np.ascontiguousarray(counts, np.int64)
    dev = _device(group)
    t = torch.from_numpy(np.ascontiguousarray(counts, np.int64)).to(dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()


LocalExtrema = Callable[[List[int]], Tuple[np.ndarray, np.ndarray]]
LocalHist = Callable[[List[int], np.ndarray, int], np.ndarray]


def sharded_collect_stats(edges: List[int], n_total: int, bins: int,
                          local_extrema: LocalExtrema, local_hist: LocalHist,
                          group=None) -> Dict[int, dict]:
    """collect_stats over all ranks' shards (reference calibration.cpp:37-115):
    pass 1 local extrema -> all-reduce -> absmax = max(|min|, |max|) -> pass 2
    local histograms against the global absmax -> all-reduce(SUM)."""
    lo, hi = local_extrema(edges)
    lo, hi = allreduce_extrema(lo, hi, group)
    absmax = np.maximum(np.abs(lo), np.abs(hi))
    counts = allreduce_counts(local_hist(edges, absmax, bins), group).reshape(len(edges), bins)
    return {k: {"min": float(lo[i]), "max": float(hi[i]), "absmax": float(absmax[i]),
                "sample_count": n_total, "counts": counts[i]} for i, k in enumerate(edges)}


class ShardedEvaluator:
    """loss(c) = 1 - sum_r same_r(c) / N over ranks (reference search.cpp:421-428);
    one all-reduce per candidate batch.  Every rank runs the same deterministic
    search on the same losses, so the search decisions agree across ranks."""

    def __init__(self, local_counts: Callable[[List[List[int]]], np.ndarray], n_total: int,
                 group=None):
        self.local_counts = local_counts
        self.n_total = n_total
        self.group = group

    def losses(self, cands: List[List[int]]) -> np.ndarray:
        same = allreduce_counts(np.asarray(self.local_counts(cands), np.int64), self.group)
        return 1.0 - same.astype(np.float64) / float(self.n_total)

    def loss(self, cand: List[int]) -> float:
        return float(self.losses([cand])[0])


@dataclass
class B200Local:
    """Per-rank compute through the B200 library's C-ABI on this rank's shard."""
    q: Q.Quantc
    graph: "Q.Graph"
    shard: "Q.Dataset"

    def extrema(self, edges: List[int]):
        L = self.q.lib
        L.qc_collect_extrema.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int), C.c_size_t,
                                         C.POINTER(C.c_double), C.POINTER(C.c_double)]
        e = np.asarray(edges, np.int32)
        lo = np.zeros(len(edges), np.float64)
        hi = np.zeros(len(edges), np.float64)
        self.q.check(L.qc_collect_extrema(self.graph.h, self.shard.h,
                                          e.ctypes.data_as(C.POINTER(C.c_int)), len(e),
                                          lo.ctypes.data_as(C.POINTER(C.c_double)),
                                          hi.ctypes.data_as(C.POINTER(C.c_double))))
        return lo, hi

    def histograms(self, edges: List[int], absmax: np.ndarray, bins: int) -> np.ndarray:
        L = self.q.lib
        L.qc_collect_histograms.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int),
                                            C.c_size_t, C.POINTER(C.c_double), C.c_int,
                                            C.POINTER(C.c_int64)]
        e = np.asarray(edges, np.int32)
        a = np.ascontiguousarray(absmax, np.float64)
        out = np.zeros(len(edges) * bins, np.int64)
        self.q.check(L.qc_collect_histograms(self.graph.h, self.shard.h,
                                             e.ctypes.data_as(C.POINTER(C.c_int)), len(e),
                                             a.ctypes.data_as(C.POINTER(C.c_double)), bins,
                                             out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out

    @staticmethod
    def agreement(q: Q.Quantc, ev: "Q.CandidateEvaluator"):
        L = q.lib
        L.qc_evaluator_agreement.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.c_size_t,
                                             C.c_size_t, C.POINTER(C.c_int64)]

        def counts(cands: List[List[int]]) -> np.ndarray:
            a = np.ascontiguousarray(np.asarray(cands, np.int32))
            out = np.zeros(a.shape[0], np.int64)
            q.check(L.qc_evaluator_agreement(ev.h, a.ctypes.data_as(C.POINTER(C.c_int)),
                                             a.shape[0], a.shape[1],
                                             out.ctypes.data_as(C.POINTER(C.c_int64))))
            return out
        return counts


def stats_handle(q: Q.Quantc, per_edge: Dict[int, dict]) -> "Q.CalibrationStats":
    """Merged statistics as a quantc CalibrationStats handle (for
    estimate_thresholds / CandidateEvaluator on every rank)."""
    return q.make_stats(per_edge)
