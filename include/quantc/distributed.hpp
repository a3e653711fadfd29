// quantc/distributed.hpp — the calibrate-and-search hot path over several
// GPUs, one process per GPU (B200 extension).
//
// The reference parallelises only over samples inside one process
// (calibration.cpp:68,95, interpreter.cpp:546) and merges per-sample partials
// associatively.  Here the unit is a rank:
//
//   collect_stats(g, shard, comm)       calibration images sharded; extrema
//                                       all-reduced between the passes,
//                                       histograms after (exact)
//   sample_sharded_losses(ev, comm)     each rank's evaluator holds its own
//                                       calibration shard; per-candidate
//                                       agreement counts are all-reduced
//   candidate_sharded_losses(ev, comm)  every rank holds the full calibration
//                                       set; a candidate batch is split over
//                                       ranks and the losses all-gathered
//
// Both loss functions plug into the *_batched searches (search.hpp): every
// rank runs the same deterministic search on the same losses, so all ranks
// reach the identical SearchResult — the one a single process computes.
#pragma once

#include <vector>

#include "quantc/calibration.hpp"
#include "quantc/comm.hpp"
#include "quantc/search.hpp"

namespace quantc {

// collect_stats over every rank's shard (reference calibration.cpp:37-115).
// `shard` is this rank's samples (may be empty on some ranks, not on all);
// EdgeStats::sample_count is the global sample count.  Bit-identical to
// collect_stats over the concatenated shards.
CalibrationStats collect_stats(const Graph& g, const Dataset& shard, Communicator& comm,
                               int bins = kDefaultHistogramBins,
                               const std::vector<int>& edge_indices = {});

// loss(c) = 1 - sum_r same_r(c) / sum_r N_r.  `ev` was built on this rank's
// calibration shard; one all-reduce of the batch's counts per call.
BatchLossFn sample_sharded_losses(const CandidateEvaluator& ev, Communicator& comm);

// Rank r evaluates its contiguous share of each candidate batch on the full
// calibration set `ev` holds; losses are all-gathered (no per-candidate
// communication beyond one gather per batch).
BatchLossFn candidate_sharded_losses(const CandidateEvaluator& ev, Communicator& comm);

// The candidate split over any per-rank batch loss: rank r calls `local` on
// its contiguous share of every batch only.  Errors on any rank surface on
// every rank after the gather (lowest failing rank's message).
BatchLossFn shard_candidates(BatchLossFn local, Communicator& comm);

}  // namespace quantc
