// quantc — command-line pipeline driver (cli module; the
// reference ships no implementation).  File-mediated phases:
//
//   quantc calibrate -m g.json -s hw.json -d data.json [--method max|quantile|kl]
//                    [--q 0.99] [--kl-bits 8] [--pow2] [--bins 2048] -o stats.json
//   quantc search    -m g.json -s hw.json -d data.json --stats stats.json
//                    [--method greedy|anneal|random|exhaustive] [--rounds 1] [--tol 0]
//                    [--seed 0] [--min-bit 4] [--steps 1000] [--t0 0.1] [--decay 0.995]
//                    [--n 100] [--cap 100000] [--threshold max|quantile|kl] [--q 0.99]
//                    [--kl-bits 8] [--pow2] -o strategy.json [--trace trace.jsonl]
//   quantc realize   -m g.json -s hw.json --strategy strategy.json -o realized.json
//   quantc eval      -a a.json -b b.json -d data.json
//
// Exit codes: 0 success, 1 usage, 2 validation (parse, file,
// fingerprint), 3 runtime.  Every command is deterministic given its inputs
// and flags.  The candidate losses run on the GPU engine (CandidateEvaluator
// batch seam, four candidates per grouped launch through the batched search).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "quantc/calibration.hpp"
#include "quantc/hwspec.hpp"
#include "quantc/interpreter.hpp"
#include "quantc/realize.hpp"
#include "quantc/search.hpp"
#include "quantc/serialize.hpp"
#include "quantc/topology.hpp"

using namespace quantc;

namespace {

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Invalid : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::string cmd;
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string get(const std::string& k, const std::string& dflt = "") const {
    auto it = kv.find(k);
    if (it != kv.end()) return it->second;
    if (dflt.empty()) throw Usage("missing " + k);
    return dflt;
  }
  double num(const std::string& k, double dflt) const {
    return has(k) ? std::stod(kv.at(k)) : dflt;
  }
};

Args parse(int argc, char** argv) {
  if (argc < 2) throw Usage("no command");
  Args a;
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("-", 0) != 0) throw Usage("unexpected argument " + k);
    if (k == "--pow2") {
      a.kv[k] = "1";
      continue;
    }
    if (i + 1 >= argc) throw Usage("flag " + k + " needs a value");
    a.kv[k] = argv[++i];
  }
  return a;
}

std::string path_arg(const Args& a, const std::string& shrt, const std::string& lng) {
  if (a.has(shrt)) return a.get(shrt);
  return a.get(lng);
}

std::string read_file(const std::string& p) {
  std::ifstream f(p, std::ios::binary);
  if (!f) throw Invalid("cannot read " + p);
  return std::string(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}

Graph load_model(const std::string& p) {
  try {
    return load_graph(p);
  } catch (const std::exception& e) {
    throw Invalid(std::string("model ") + p + ": " + e.what());
  }
}

HardwareSpec load_spec(const std::string& p) {
  try {
    return parse_spec(read_file(p));
  } catch (const Invalid&) {
    throw;
  } catch (const std::exception& e) {
    throw Invalid(std::string("spec ") + p + ": " + e.what());
  }
}

Dataset load_data(const std::string& p) {
  try {
    return load_dataset(p);
  } catch (const std::exception& e) {
    throw Invalid(std::string("dataset ") + p + ": " + e.what());
  }
}

ThresholdConfig threshold_config(const Args& a, const std::string& key) {
  ThresholdConfig c;
  const std::string m = a.has(key) ? a.get(key) : "quantile";
  if (m == "max") {
    c.method = ThresholdMethod::kMax;
  } else if (m == "quantile") {
    c.method = ThresholdMethod::kQuantile;
  } else if (m == "kl") {
    c.method = ThresholdMethod::kKl;
  } else {
    throw Usage("unknown threshold method " + m);
  }
  c.quantile = a.num("--q", 0.99);
  c.kl_bits = static_cast<int>(a.num("--kl-bits", 8));
  c.pow2 = a.has("--pow2");
  return c;
}

int cmd_calibrate(const Args& a) {
  const Graph g = load_model(path_arg(a, "-m", "--model"));
  const HardwareSpec spec = load_spec(path_arg(a, "-s", "--spec"));
  const Dataset d = load_data(path_arg(a, "-d", "--dataset"));
  const std::string out = path_arg(a, "-o", "--out");
  const Topology t = generate_topology(g, spec);
  CalibrationStats st = collect_stats(g, d, static_cast<int>(a.num("--bins", kDefaultHistogramBins)),
                                      simulated_edge_indices(g, t));
  st.graph_fingerprint = fingerprint_graph(g);
  st.dataset_fingerprint = fingerprint_dataset(d);
  save_stats(st, out);
  const auto thr = estimate_thresholds(st, threshold_config(a, "--method"));
  std::printf("edge\tthreshold\n");
  for (const auto& [e, v] : thr) std::printf("%d\t%.17g\n", e, v);
  return 0;
}

int cmd_search(const Args& a) {
  const Graph g = load_model(path_arg(a, "-m", "--model"));
  const HardwareSpec spec = load_spec(path_arg(a, "-s", "--spec"));
  const Dataset d = load_data(path_arg(a, "-d", "--dataset"));
  CalibrationStats st;
  try {
    st = load_stats(a.get("--stats"));
  } catch (const std::exception& e) {
    throw Invalid(std::string("stats: ") + e.what());
  }
  if (st.graph_fingerprint != 0 && st.graph_fingerprint != fingerprint_graph(g)) {
    throw Invalid("stats were collected on a different graph (fingerprint mismatch)");
  }
  if (st.dataset_fingerprint != 0 && st.dataset_fingerprint != fingerprint_dataset(d)) {
    throw Invalid("stats were collected on a different dataset (fingerprint mismatch)");
  }
  const Topology t = generate_topology(g, spec);
  const Graph sim = insert_simulated_quantize(g, t);
  const auto thr = estimate_thresholds(st, threshold_config(a, "--threshold"));
  const int min_bit = static_cast<int>(a.num("--min-bit", kDefaultMinBit));
  CandidateEvaluator ev(sim, spec, t, thr, st, d, min_bit);
  const SearchSpace& space = ev.space();
  const BatchLossFn losses = ev.batch_loss();
  const std::string method = a.has("--method") ? a.get("--method") : "greedy";
  const uint64_t seed = static_cast<uint64_t>(a.num("--seed", 0));
  SearchResult r;
  if (method == "greedy") {
    r = greedy_search_batched(space, losses, static_cast<int>(a.num("--rounds", 1)), a.num("--tol", 0.0));
  } else if (method == "anneal") {
    r = anneal_search_batched(space, losses, static_cast<int>(a.num("--steps", 1000)), a.num("--t0", 0.1),
                              a.num("--decay", 0.995), seed);
  } else if (method == "random") {
    r = random_search_batched(space, losses, static_cast<int>(a.num("--n", 100)), seed);
  } else if (method == "exhaustive") {
    r = exhaustive_search_batched(space, losses, static_cast<int64_t>(a.num("--cap", 100000)));
  } else {
    throw Usage("unknown search method " + method);
  }
  Json meta = {{"method", method}, {"best_loss", r.best_loss}, {"evaluations", r.evaluations},
               {"space_size", space_size(space).str()}};
  save_strategy(ev.strategy_for(r.best), meta, path_arg(a, "-o", "--out"));
  if (a.has("--trace")) save_trace(r.trace, a.get("--trace"));
  std::printf("final loss %.17g, evaluations %lld, space size %s\n", r.best_loss,
              static_cast<long long>(r.evaluations), space_size(space).str().c_str());
  return 0;
}

int cmd_realize(const Args& a) {
  const Graph g = load_model(path_arg(a, "-m", "--model"));
  const HardwareSpec spec = load_spec(path_arg(a, "-s", "--spec"));
  Strategy s;
  try {
    s = load_strategy(a.get("--strategy"));
  } catch (const std::exception& e) {
    throw Invalid(std::string("strategy: ") + e.what());
  }
  const Graph sim = insert_simulated_quantize(g, generate_topology(g, spec));
  const Graph r = realize(sim, s, spec);
  save_graph(r, path_arg(a, "-o", "--out"));
  std::map<std::string, int> ops;
  for (const Node& n : r.nodes()) ops[op_name(n.op)]++;
  std::printf("nodes %zu -> %zu (%+lld)\n", g.nodes().size(), r.nodes().size(),
              static_cast<long long>(r.nodes().size()) - static_cast<long long>(g.nodes().size()));
  for (const auto& [k, v] : ops) std::printf("  %s\t%d\n", k.c_str(), v);
  return 0;
}

int cmd_eval(const Args& a) {
  const Graph ga = load_model(path_arg(a, "-a", "--model-a"));
  const Graph gb = load_model(path_arg(a, "-b", "--model-b"));
  const Dataset d = load_data(path_arg(a, "-d", "--dataset"));
  int64_t agree = 0, ca = 0, cb = 0, labeled = 0;
  double mad = 0.0;
  int64_t count = 0;
  for (const Sample& s : d) {
    const Tensor ya = eval_model(ga, feed_for(ga, s)).at(0);
    const Tensor yb = eval_model(gb, feed_for(gb, s)).at(0);
    if (ya.numel() != yb.numel()) throw Invalid("output shapes differ between the two models");
    const int64_t pa = argmax_class(ya), pb = argmax_class(yb);
    agree += pa == pb;
    if (s.label) {
      ++labeled;
      ca += pa == *s.label;
      cb += pb == *s.label;
    }
    if (ya.dtype().is_float() && yb.dtype().is_float()) {
      const auto fa = ya.floats(), fb = yb.floats();
      for (size_t i = 0; i < fa.size(); ++i) {
        mad += std::abs(static_cast<double>(fa[i]) - static_cast<double>(fb[i]));
        ++count;
      }
    }
  }
  const double n = static_cast<double>(d.size());
  std::printf("top1 agreement %.6f\n", d.empty() ? 0.0 : agree / n);
  if (labeled) {
    std::printf("accuracy a %.6f b %.6f drop %.6f\n", ca / static_cast<double>(labeled),
                cb / static_cast<double>(labeled), (ca - cb) / static_cast<double>(labeled));
  }
  if (count) std::printf("mean abs output difference %.9g\n", mad / static_cast<double>(count));
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.cmd == "calibrate") return cmd_calibrate(a);
    if (a.cmd == "search") return cmd_search(a);
    if (a.cmd == "realize") return cmd_realize(a);
    if (a.cmd == "eval") return cmd_eval(a);
    throw Usage("unknown command " + a.cmd);
  } catch (const Usage& e) {
    std::fprintf(stderr, "usage error: %s\n(commands: calibrate, search, realize, eval)\n", e.what());
    return 1;
  } catch (const Invalid& e) {
    std::fprintf(stderr, "invalid input: %s\n", e.what());
    return 2;
  } catch (const IoError& e) {
    std::fprintf(stderr, "invalid input: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
}
