// calibration.cpp — statistics collection and threshold estimation on the
// GPU (reference calibration.cpp:14-234).
//
// collect_stats keeps the reference's two-pass structure (exact extrema, then
// histograms against the final absmax) but runs each pass as batched GPU
// forwards with the statistics kernels hooked onto the producing steps.  When
// the target activations of the whole calibration set fit in the memory
// budget, pass 1 keeps them resident and pass 2 reads them back instead of
// recomputing the forward (the reference recomputes, calibration.cpp:95-96;
// the values are identical either way).  Constant (weight) edges are reduced
// once and their counts scaled by the sample count — the reference
// re-histograms the same tensor for every sample, so the counts are equal.
#include "quantc/calibration.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <limits>
#include <memory>
#include <mutex>
#include <unordered_map>

#include "dataset.hpp"
#include "engine.hpp"
#include "quantc/device.hpp"
#include "quantc/distributed.hpp"

namespace quantc {

namespace {
cudaStream_t S() { return static_cast<cudaStream_t>(device::stream()); }
void ok(cudaError_t e) {
  if (e != cudaSuccess) throw DeviceError(cudaGetErrorString(e));
}
}  // namespace

int64_t EdgeStats::total_count() const {
  int64_t n = 0;
  for (int64_t c : counts) n += c;
  return n;
}

double EdgeStats::bin_upper_edge(int i) const {
  return absmax * (static_cast<double>(i + 1) / static_cast<double>(counts.size()));
}

CalibrationStats collect_stats(const Graph& g, const Dataset& dataset, int bins,
                               const std::vector<int>& edge_indices, int workers) {
  (void)workers;
  if (dataset.empty()) throw CalibrationError("calibration dataset is empty");
  if (bins < 2) throw CalibrationError("histogram needs at least 2 bins");
  const std::vector<Edge> edges = edge_order(g);
  std::vector<int> targets = edge_indices;
  if (targets.empty()) {
    for (size_t k = 0; k < edges.size(); ++k) targets.push_back(static_cast<int>(k));
  }
  for (int k : targets) {
    if (k < 0 || k >= static_cast<int>(edges.size())) {
      throw CalibrationError("edge index " + std::to_string(k) + " out of range");
    }
  }

  engine::Plan plan(g);
  gpu::DeviceDataset dd(g, dataset);
  const int64_t N = dd.size();

  // one statistics slot per distinct producer step
  std::unordered_map<int, int> slot_of_step;
  std::vector<int> slot_step;
  std::vector<int> edge_slot(targets.size());
  for (size_t t = 0; t < targets.size(); ++t) {
    const int step = plan.step_of(edges[static_cast<size_t>(targets[t])].src.node);
    auto it = slot_of_step.find(step);
    if (it == slot_of_step.end()) {
      it = slot_of_step.emplace(step, static_cast<int>(slot_step.size())).first;
      slot_step.push_back(step);
    }
    edge_slot[t] = it->second;
  }
  const int n_slots = static_cast<int>(slot_step.size());

  auto keys = engine::device_alloc(static_cast<size_t>(n_slots) * 16);
  auto* k64 = static_cast<unsigned long long*>(keys.get());
  kern::minmax_init(k64, n_slots, S());

  // resident-activation cache for pass 2
  int64_t per_sample_bytes = 0;
  for (int st : slot_step) {
    if (plan.batched(st)) per_sample_bytes += shape_numel(plan.shape(st)) * 4;
  }
  const bool cache = per_sample_bytes * N <= static_cast<int64_t>(device::memory_budget_bytes());
  std::vector<std::vector<std::pair<int, engine::DevTensor>>> cached;  // per batch

  const int batch = plan.batch_for(N);
  using Hook = std::function<void(int step, const engine::DevTensor&, int b, int64_t bi)>;
  auto forward = [&](const Hook& hook) {
    int64_t bi = 0;
    for (int64_t s0 = 0; s0 < N; s0 += batch, ++bi) {
      const int b = static_cast<int>(std::min<int64_t>(batch, N - s0));
      engine::RunSpec spec;
      spec.batch = b;
      for (size_t k = 0; k < dd.num_inputs(); ++k) spec.inputs.push_back(dd.input(k, s0));
      spec.on_value = [&, b, bi](int step, const engine::DevTensor& v) {
        if (slot_of_step.count(step)) hook(step, v, b, bi);
      };
      engine::run(plan, spec);
    }
  };
  auto require_float = [](const engine::DevTensor& v) {
    if (!v.dtype.is_float()) throw std::logic_error("floats() on " + v.dtype.name() + " tensor");
  };

  // pass 1: exact extrema (calibration.cpp:62-91)
  std::vector<int> batch_size_of;
  forward([&](int step, const engine::DevTensor& v, int b, int64_t bi) {
    require_float(v);
    const int slot = slot_of_step.at(step);
    if (v.batched || bi == 0) kern::minmax_accumulate(v.f(), v.numel(b), k64 + 2 * slot, S());
    if (cache) {
      if (static_cast<int64_t>(cached.size()) <= bi) {
        cached.resize(static_cast<size_t>(bi) + 1);
        batch_size_of.resize(static_cast<size_t>(bi) + 1);
      }
      batch_size_of[static_cast<size_t>(bi)] = b;
      if (v.batched || bi == 0) cached[static_cast<size_t>(bi)].push_back({step, v});
    }
  });
  std::vector<double> mm(static_cast<size_t>(n_slots) * 2);
  {
    auto dmm = engine::device_alloc(mm.size() * 8);
    kern::minmax_decode(k64, static_cast<double*>(dmm.get()), n_slots, S());
    ok(cudaMemcpyAsync(mm.data(), dmm.get(), mm.size() * 8, cudaMemcpyDeviceToHost, S()));
    device::synchronize();
  }
  std::vector<double> absmax(static_cast<size_t>(n_slots));
  for (int s = 0; s < n_slots; ++s) {
    absmax[static_cast<size_t>(s)] =
        std::max(std::fabs(mm[2 * static_cast<size_t>(s)]), std::fabs(mm[2 * static_cast<size_t>(s) + 1]));
  }

  // pass 2: histograms against the final absmax (calibration.cpp:93-113)
  auto counts = engine::device_alloc(static_cast<size_t>(n_slots) * bins * 8);
  ok(cudaMemsetAsync(counts.get(), 0, static_cast<size_t>(n_slots) * bins * 8, S()));
  auto* c64 = static_cast<unsigned long long*>(counts.get());
  auto hist = [&](int step, const engine::DevTensor& v, int b, int64_t bi) {
    const int slot = slot_of_step.at(step);
    if (v.batched) {
      kern::histogram_accumulate(v.f(), v.numel(b), absmax[static_cast<size_t>(slot)], bins,
                                 c64 + static_cast<int64_t>(slot) * bins, 1ull, S());
    } else if (bi == 0) {
      kern::histogram_accumulate(v.f(), v.numel(b), absmax[static_cast<size_t>(slot)], bins,
                                 c64 + static_cast<int64_t>(slot) * bins,
                                 static_cast<unsigned long long>(N), S());
    }
  };
  if (cache) {
    for (size_t bi = 0; bi < cached.size(); ++bi) {
      for (auto& [step, v] : cached[bi]) hist(step, v, batch_size_of[bi], static_cast<int64_t>(bi));
      cached[bi].clear();
    }
  } else {
    forward(hist);
  }
  std::vector<int64_t> hc(static_cast<size_t>(n_slots) * bins);
  ok(cudaMemcpyAsync(hc.data(), counts.get(), hc.size() * 8, cudaMemcpyDeviceToHost, S()));
  device::synchronize();

  CalibrationStats stats;
  for (size_t t = 0; t < targets.size(); ++t) {
    const size_t s = static_cast<size_t>(edge_slot[t]);
    EdgeStats e;
    e.min = mm[2 * s];
    e.max = mm[2 * s + 1];
    e.absmax = absmax[s];
    e.sample_count = N;
    e.counts.assign(hc.begin() + static_cast<int64_t>(s) * bins,
                    hc.begin() + static_cast<int64_t>(s + 1) * bins);
    stats.per_edge[targets[t]] = std::move(e);
  }
  return stats;
}

namespace {

// Shared driver of the sharded passes: batched forwards over `ds` with
// `hook(slot, value, batch, batch_index)` on every target producer step.
struct ShardPasses {
  engine::PlanLease lease;  // weights stay resident across the two passes
  const engine::Plan& plan;
  gpu::DeviceDataset dd;
  std::unordered_map<int, int> slot_of_step;
  std::vector<int> edge_slot;
  int n_slots = 0;

  ShardPasses(const Graph& g, const Dataset& ds, const std::vector<int>& edges_idx)
      : lease(engine::lease_plan(g)), plan(lease.plan()), dd(g, ds) {
    const std::vector<Edge> edges = edge_order(g);
    for (int k : edges_idx) {
      if (k < 0 || k >= static_cast<int>(edges.size())) {
        throw CalibrationError("edge index " + std::to_string(k) + " out of range");
      }
      const int step = plan.step_of(edges[static_cast<size_t>(k)].src.node);
      auto it = slot_of_step.find(step);
      if (it == slot_of_step.end()) it = slot_of_step.emplace(step, n_slots++).first;
      edge_slot.push_back(it->second);
    }
  }

  // device bytes of the targets' batched activations for the whole shard
  int64_t resident_bytes() const {
    int64_t per = 0;
    for (const auto& [step, slot] : slot_of_step) {
      if (plan.batched(step)) per += shape_numel(plan.shape(step)) * 4;
    }
    return per * dd.size();
  }

  template <typename Hook>
  void forward(Hook&& hook) {
    const int64_t N = dd.size();
    const int batch = plan.batch_for(N);
    static const bool hprof = std::getenv("QUANTC_HOST_PROF") != nullptr;
    if (hprof) {
      std::fprintf(stderr, "ShardPasses::forward N %lld batch %d budget %zu\n",
                   static_cast<long long>(N), batch, device::memory_budget_bytes());
    }
    int64_t bi = 0;
    for (int64_t s0 = 0; s0 < N; s0 += batch, ++bi) {
      const int b = static_cast<int>(std::min<int64_t>(batch, N - s0));
      engine::RunSpec spec;
      spec.batch = b;
      for (size_t k = 0; k < dd.num_inputs(); ++k) spec.inputs.push_back(dd.input(k, s0));
      spec.on_value = [&, b, bi](int step, const engine::DevTensor& v) {
        auto it = slot_of_step.find(step);
        if (it == slot_of_step.end()) return;
        if (!v.dtype.is_float()) throw std::logic_error("floats() on " + v.dtype.name() + " tensor");
        hook(it->second, v, b, bi);
      };
      const auto tr = std::chrono::steady_clock::now();
      engine::run(plan, spec);
      if (hprof) {
        const double host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tr).count();
        device::synchronize();
        std::fprintf(stderr, "  run batch %d: host %.1f ms, +sync %.1f ms\n", b, host_ms,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tr).count());
      }
    }
  }
};

// Activations pass 1 keeps resident for pass 2 (when the whole shard's
// target activations fit the memory budget), exactly like collect_stats'
// single-call cache: pass 2 then reads them instead of re-running the forward.
struct PassCache {
  std::vector<int> edge_slot;
  int n_slots = 0;
  std::vector<std::vector<std::pair<int, engine::DevTensor>>> batches;  // (slot, value)
  std::vector<int> batch_size;
};

// Pass 1 over one shard: exact per-edge extrema (calibration.cpp:62-91).
std::unique_ptr<PassCache> pass_extrema(ShardPasses& sp, bool keep, std::vector<double>* mins,
                                        std::vector<double>* maxs) {
  auto keys = engine::device_alloc(static_cast<size_t>(sp.n_slots) * 16 + 16);
  auto* k64 = static_cast<unsigned long long*>(keys.get());
  kern::minmax_init(k64, sp.n_slots, S());
  std::unique_ptr<PassCache> h;
  if (keep && sp.resident_bytes() <= static_cast<int64_t>(device::memory_budget_bytes())) {
    // grow the stream-ordered pool once for the retained activations (plus a
    // batch's transient working set) instead of in many small mappings
    device::pool_reserve(static_cast<size_t>(sp.resident_bytes()) * 5 / 4);
    h = std::make_unique<PassCache>();
    h->edge_slot = sp.edge_slot;
    h->n_slots = sp.n_slots;
  }
  sp.forward([&](int slot, const engine::DevTensor& v, int b, int64_t bi) {
    if (v.batched || bi == 0) kern::minmax_accumulate(v.f(), v.numel(b), k64 + 2 * slot, S());
    if (h && (v.batched || bi == 0)) {
      if (static_cast<int64_t>(h->batches.size()) <= bi) {
        h->batches.resize(static_cast<size_t>(bi) + 1);
        h->batch_size.resize(static_cast<size_t>(bi) + 1);
      }
      h->batch_size[static_cast<size_t>(bi)] = b;
      h->batches[static_cast<size_t>(bi)].push_back({slot, v});
    }
  });
  std::vector<double> mm(static_cast<size_t>(sp.n_slots) * 2);
  auto dmm = engine::device_alloc(mm.size() * 8 + 16);
  kern::minmax_decode(k64, static_cast<double*>(dmm.get()), sp.n_slots, S());
  ok(cudaMemcpyAsync(mm.data(), dmm.get(), mm.size() * 8, cudaMemcpyDeviceToHost, S()));
  device::synchronize();
  mins->clear();
  maxs->clear();
  for (int s : sp.edge_slot) {
    mins->push_back(mm[2 * static_cast<size_t>(s)]);
    maxs->push_back(mm[2 * static_cast<size_t>(s) + 1]);
  }
  return h;
}

// Pass 2 over one shard: histograms against the given (global) absmax per
// edge (calibration.cpp:93-113).  From the pass-1 cache when there is one,
// else by a fresh forward of `sp`.  Constant edges are counted once and
// scaled by the shard's sample count N.
void pass_histograms(ShardPasses* sp, PassCache* cache, const std::vector<int>& edges,
                     const std::vector<double>& absmax, int bins, int64_t N,
                     std::vector<int64_t>* counts) {
  const int n_slots = cache ? cache->n_slots : sp->n_slots;
  const std::vector<int>& edge_slot = cache ? cache->edge_slot : sp->edge_slot;
  std::vector<double> slot_absmax(static_cast<size_t>(n_slots), 0.0);
  for (size_t t = 0; t < edges.size(); ++t) slot_absmax[static_cast<size_t>(edge_slot[t])] = absmax[t];
  auto dc = engine::device_alloc(static_cast<size_t>(n_slots) * bins * 8 + 16);
  ok(cudaMemsetAsync(dc.get(), 0, static_cast<size_t>(n_slots) * bins * 8, S()));
  auto* c64 = static_cast<unsigned long long*>(dc.get());
  auto hist = [&](int slot, const engine::DevTensor& v, int b, int64_t bi) {
    if (v.batched) {
      kern::histogram_accumulate(v.f(), v.numel(b), slot_absmax[static_cast<size_t>(slot)], bins,
                                 c64 + static_cast<int64_t>(slot) * bins, 1ull, S());
    } else if (bi == 0) {
      kern::histogram_accumulate(v.f(), v.numel(b), slot_absmax[static_cast<size_t>(slot)], bins,
                                 c64 + static_cast<int64_t>(slot) * bins,
                                 static_cast<unsigned long long>(N), S());
    }
  };
  if (cache) {
    for (size_t bi = 0; bi < cache->batches.size(); ++bi) {
      for (auto& [slot, v] : cache->batches[bi]) {
        hist(slot, v, cache->batch_size[bi], static_cast<int64_t>(bi));
      }
    }
  } else {
    sp->forward(hist);
  }
  std::vector<int64_t> hc(static_cast<size_t>(n_slots) * bins);
  ok(cudaMemcpyAsync(hc.data(), dc.get(), hc.size() * 8, cudaMemcpyDeviceToHost, S()));
  device::synchronize();
  counts->clear();
  for (int s : edge_slot) {
    counts->insert(counts->end(), hc.begin() + static_cast<int64_t>(s) * bins,
                   hc.begin() + static_cast<int64_t>(s + 1) * bins);
  }
}

// Pass-1 -> pass-2 handoff between the two sharded C-ABI calls
// (qc_collect_extrema / qc_collect_histograms, between which the caller
// all-reduces the extrema).  Keyed on the graph's uid and a caller-supplied
// shard key (the C-ABI dataset handle's uid): never on addresses, which the
// allocator can reuse.  Key 0 disables the handoff (pass 2 recomputes).
struct Handoff {
  uint64_t graph_uid = 0;
  uint64_t shard_key = 0;
  std::vector<int> edges;
  std::unique_ptr<PassCache> cache;
};
std::mutex g_handoff_mu;
std::unique_ptr<Handoff> g_handoff;

}  // namespace

void collect_extrema(const Graph& g, const Dataset& shard, const std::vector<int>& edges,
                     std::vector<double>* mins, std::vector<double>* maxs, uint64_t shard_key) {
  if (shard.empty()) throw CalibrationError("calibration dataset is empty");
  ShardPasses sp(g, shard, edges);
  {
    std::lock_guard<std::mutex> lk(g_handoff_mu);
    g_handoff.reset();  // a new pass 1 supersedes any unconsumed handoff
  }
  auto cache = pass_extrema(sp, shard_key != 0, mins, maxs);
  if (cache) {
    auto h = std::make_unique<Handoff>();
    h->graph_uid = g.uid();
    h->shard_key = shard_key;
    h->edges = edges;
    h->cache = std::move(cache);
    std::lock_guard<std::mutex> lk(g_handoff_mu);
    g_handoff = std::move(h);
  }
}

void collect_histograms(const Graph& g, const Dataset& shard, const std::vector<int>& edges,
                        const std::vector<double>& absmax, int bins,
                        std::vector<int64_t>* counts, uint64_t shard_key) {
  if (shard.empty()) throw CalibrationError("calibration dataset is empty");
  if (bins < 2) throw CalibrationError("histogram needs at least 2 bins");
  if (absmax.size() != edges.size()) throw std::invalid_argument("absmax per edge required");
  std::unique_ptr<Handoff> h;
  {
    std::lock_guard<std::mutex> lk(g_handoff_mu);
    if (shard_key != 0 && g_handoff && g_handoff->graph_uid == g.uid() &&
        g_handoff->shard_key == shard_key && g_handoff->edges == edges) {
      h = std::move(g_handoff);
    }
    g_handoff.reset();
  }
  std::unique_ptr<ShardPasses> sp;
  if (!h) sp = std::make_unique<ShardPasses>(g, shard, edges);
  pass_histograms(sp.get(), h ? h->cache.get() : nullptr, edges, absmax, bins,
                  static_cast<int64_t>(shard.size()), counts);
}

// Distributed collect_stats (quantc/distributed.hpp): pass 1 on this rank's
// shard -> all-reduce MIN / MAX -> absmax -> pass 2 against the global absmax
// -> all-reduce SUM.  Every merge is exact, so the result equals
// collect_stats over the concatenated shards.  An empty shard contributes the
// identities (+inf / -inf, zero counts).
CalibrationStats collect_stats(const Graph& g, const Dataset& shard, Communicator& comm, int bins,
                               const std::vector<int>& edge_indices) {
  if (bins < 2) throw CalibrationError("histogram needs at least 2 bins");
  const size_t n_edges = edge_order(g).size();
  std::vector<int> targets = edge_indices;
  if (targets.empty()) {
    for (size_t k = 0; k < n_edges; ++k) targets.push_back(static_cast<int>(k));
  }
  for (int k : targets) {
    if (k < 0 || k >= static_cast<int>(n_edges)) {
      throw CalibrationError("edge index " + std::to_string(k) + " out of range");
    }
  }
  int64_t n_total = static_cast<int64_t>(shard.size());
  comm.allreduce_sum(&n_total, 1);
  if (n_total == 0) throw CalibrationError("calibration dataset is empty");
  const size_t T = targets.size();
  std::vector<double> lo(T, std::numeric_limits<double>::infinity());
  std::vector<double> hi(T, -std::numeric_limits<double>::infinity());
  std::unique_ptr<ShardPasses> sp;
  std::unique_ptr<PassCache> cache;
  if (!shard.empty()) {
    sp = std::make_unique<ShardPasses>(g, shard, targets);
    cache = pass_extrema(*sp, true, &lo, &hi);
  }
  comm.allreduce_min(lo.data(), T);
  comm.allreduce_max(hi.data(), T);
  std::vector<double> absmax(T);
  for (size_t t = 0; t < T; ++t) absmax[t] = std::max(std::fabs(lo[t]), std::fabs(hi[t]));
  std::vector<int64_t> counts(T * static_cast<size_t>(bins), 0);
  if (!shard.empty()) {
    pass_histograms(sp.get(), cache.get(), targets, absmax, bins,
                    static_cast<int64_t>(shard.size()), &counts);
  }
  cache.reset();
  comm.allreduce_sum(counts.data(), counts.size());
  CalibrationStats stats;
  for (size_t t = 0; t < T; ++t) {
    EdgeStats e;
    e.min = lo[t];
    e.max = hi[t];
    e.absmax = absmax[t];
    e.sample_count = n_total;
    e.counts.assign(counts.begin() + static_cast<int64_t>(t) * bins,
                    counts.begin() + static_cast<int64_t>(t + 1) * bins);
    stats.per_edge[targets[t]] = std::move(e);
  }
  return stats;
}

double threshold_max(const EdgeStats& stats) {
  return stats.absmax > 0.0 ? stats.absmax : kDegenerateThreshold;
}

double threshold_quantile(const EdgeStats& stats, double q) {
  if (!(q > 0.0) || q > 1.0) throw CalibrationError("quantile must be in (0, 1]");
  if (stats.absmax <= 0.0) return kDegenerateThreshold;
  const int64_t total = stats.total_count();
  if (total == 0) throw CalibrationError("histogram is empty");
  int64_t cum = 0;
  for (size_t b = 0; b < stats.counts.size(); ++b) {
    cum += stats.counts[b];
    if (static_cast<double>(cum) >= q * static_cast<double>(total)) {
      return stats.bin_upper_edge(static_cast<int>(b));
    }
  }
  return stats.absmax;
}

namespace {

// Validation + degenerate handling of reference calibration.cpp:161-169.
// Returns true when the edge needs the KL sweep.
bool kl_precheck(const EdgeStats& s, int target_bit, double* degenerate) {
  if (target_bit < 1 || target_bit > 16) throw CalibrationError("target_bit out of range");
  const int bins = static_cast<int>(s.counts.size());
  if (bins < (1 << target_bit)) {
    throw CalibrationError("histogram has fewer bins than 2^target_bit levels");
  }
  if (s.total_count() == 0) throw CalibrationError("histogram is empty");
  if (s.absmax <= 0.0) {
    *degenerate = kDegenerateThreshold;
    return false;
  }
  return true;
}

// Runs the device KL sweep over a group of edges with equal bin counts.
std::vector<int> kl_best_indices(const std::vector<const EdgeStats*>& es, int target_bit) {
  const int bins = static_cast<int>(es[0]->counts.size());
  std::vector<int64_t> flat;
  flat.reserve(es.size() * static_cast<size_t>(bins));
  for (const EdgeStats* e : es) flat.insert(flat.end(), e->counts.begin(), e->counts.end());
  auto dc = engine::device_alloc(flat.size() * 8);
  ok(cudaMemcpyAsync(dc.get(), flat.data(), flat.size() * 8, cudaMemcpyHostToDevice, S()));
  auto di = engine::device_alloc(es.size() * 4);
  auto dk = engine::device_alloc(es.size() * 8);
  kern::kl_sweep(static_cast<const int64_t*>(dc.get()), static_cast<int>(es.size()), bins,
                 target_bit, static_cast<int*>(di.get()), static_cast<double*>(dk.get()), S());
  std::vector<int> best(es.size());
  ok(cudaMemcpyAsync(best.data(), di.get(), best.size() * 4, cudaMemcpyDeviceToHost, S()));
  device::synchronize();
  return best;
}

}  // namespace

double threshold_kl(const EdgeStats& stats, int target_bit) {
  double degenerate = 0.0;
  if (!kl_precheck(stats, target_bit, &degenerate)) return degenerate;
  const int best = kl_best_indices({&stats}, target_bit)[0];
  return stats.absmax *
         (static_cast<double>(best) / static_cast<double>(stats.counts.size()));
}

double round_pow2(double threshold) {
  if (!(threshold > 0.0)) throw CalibrationError("round_pow2 needs a positive threshold");
  return std::exp2(std::floor(std::log2(threshold) + 0.5));
}

std::map<int, double> estimate_thresholds(const CalibrationStats& stats,
                                          const ThresholdConfig& config) {
  std::map<int, double> result;
  if (config.method == ThresholdMethod::kKl) {
    // validate in edge order (first failing edge throws, like the reference),
    // then sweep all remaining edges in one launch per bin count
    std::map<int, std::vector<std::pair<int, const EdgeStats*>>> by_bins;
    for (const auto& [k, e] : stats.per_edge) {
      double deg = 0.0;
      if (kl_precheck(e, config.kl_bits, &deg)) {
        by_bins[static_cast<int>(e.counts.size())].push_back({k, &e});
      } else {
        result[k] = deg;
      }
    }
    for (const auto& [bins, group] : by_bins) {
      std::vector<const EdgeStats*> es;
      for (const auto& kv : group) es.push_back(kv.second);
      std::vector<int> best = kl_best_indices(es, config.kl_bits);
      for (size_t j = 0; j < group.size(); ++j) {
        result[group[j].first] =
            group[j].second->absmax * (static_cast<double>(best[j]) / static_cast<double>(bins));
      }
    }
  } else {
    for (const auto& [k, e] : stats.per_edge) {
      result[k] = config.method == ThresholdMethod::kMax ? threshold_max(e)
                  : e.absmax > 0.0 ? threshold_quantile(e, config.quantile)
                                   : kDegenerateThreshold;
    }
  }
  if (config.pow2) {
    for (auto& [k, t] : result) t = round_pow2(t);
  }
  return result;
}

}  // namespace quantc
