// distributed.cpp — the search's two multi-rank loss functions
// (quantc/distributed.hpp).  The distributed collect_stats lives next to the
// pass helpers it shares with the single-process path (calibration.cpp).
#include "quantc/distributed.hpp"

#include <cmath>
#include <limits>
#include <string>

namespace quantc {

BatchLossFn sample_sharded_losses(const CandidateEvaluator& ev, Communicator& comm) {
  int64_t n_total = static_cast<int64_t>(ev.reference_predictions().size());
  comm.allreduce_sum(&n_total, 1);
  if (n_total == 0) throw SearchError("calibration set is empty on every rank");
  return [&ev, &comm, n_total](std::span<const Candidate> cs) {
    // bind errors are deterministic (same candidates, same tables on every
    // rank), so every rank throws before the collective alike
    std::vector<int64_t> same = ev.agreement_counts(cs);
    comm.allreduce_sum(same.data(), same.size());
    std::vector<double> out(same.size());
    for (size_t i = 0; i < same.size(); ++i) {
      out[i] = 1.0 - static_cast<double>(same[i]) / static_cast<double>(n_total);
    }
    return out;
  };
}

BatchLossFn candidate_sharded_losses(const CandidateEvaluator& ev, Communicator& comm) {
  return shard_candidates(ev.batch_loss(), comm);
}

BatchLossFn shard_candidates(BatchLossFn local, Communicator& comm) {
  return [local = std::move(local), &comm](std::span<const Candidate> cs) {
    const int R = comm.size();
    const int64_t n = static_cast<int64_t>(cs.size());
    const auto [first, last] = shard_range(n, comm.rank(), R);
    const int64_t share = (n + R - 1) / R;  // gather width (ranks pad to it)
    // slot 0: status (-1 ok, else the failing global candidate index)
    std::vector<double> send(static_cast<size_t>(share) + 1,
                             std::numeric_limits<double>::quiet_NaN());
    send[0] = -1.0;
    std::string why;
    try {
      if (last > first) {
        const std::vector<double> l = local(cs.subspan(static_cast<size_t>(first),
                                                       static_cast<size_t>(last - first)));
        if (l.size() != static_cast<size_t>(last - first)) {
          throw SearchError("batched loss returned the wrong count");
        }
        std::copy(l.begin(), l.end(), send.begin() + 1);
      }
    } catch (const std::exception& e) {
      // report after the gather so no rank is left waiting in it
      why = e.what();
      send[0] = static_cast<double>(first);
    }
    std::vector<double> all(send.size() * static_cast<size_t>(R));
    comm.allgather(send.data(), send.size(), all.data());
    std::vector<double> out;
    out.reserve(static_cast<size_t>(n));
    for (int r = 0; r < R; ++r) {
      const double* blk = all.data() + static_cast<size_t>(r) * send.size();
      if (blk[0] >= 0.0) {
        throw SearchError(r == comm.rank() ? why
                                           : "candidate batch failed on rank " + std::to_string(r) +
                                                 " (from candidate " +
                                                 std::to_string(static_cast<int64_t>(blk[0])) + ")");
      }
      const auto [f, l] = shard_range(n, r, R);
      out.insert(out.end(), blk + 1, blk + 1 + (l - f));
    }
    return out;
  };
}

}  // namespace quantc
