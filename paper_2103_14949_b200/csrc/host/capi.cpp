// capi.cpp — the flat C-ABI (include/quantc_capi.h) over the quantc C++ API.
//
// This translation unit uses ONLY the public quantc headers, so it compiles
// unchanged against
//   * this repo's B200 implementation (include/quantc/*.hpp), and
//   * the reference sources (/root/reference/proj/include), see oracle/Makefile.
// That double build is the executable proof that the boundary is a drop-in:
// the same binding code drives both.  Reference interfaces are cited per entry
// point in include/quantc_capi.h.
#include "quantc_capi.h"

#include <atomic>
#include <cstdlib>
#include <functional>
#include <map>
#include <span>
#include <cstring>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "quantc/calibration.hpp"
#include "quantc/dtype.hpp"
#include "quantc/graph.hpp"
#include "quantc/hwspec.hpp"
#include "quantc/interpreter.hpp"
#include "quantc/search.hpp"
#include "quantc/simulate.hpp"
#include "quantc/tensor.hpp"
#include "quantc/topology.hpp"
#ifdef QUANTC_B200
#include "quantc/device.hpp"
#include "quantc/distributed.hpp"
#include "quantc/fixtures.hpp"
#include "quantc/serialize.hpp"
#include "quantc_files.h"
#include "quantc_cuda.h"
#include "engine.hpp"
#endif

using namespace quantc;

struct qc_graph {
  std::shared_ptr<Graph> g;
};
struct qc_spec {
  std::shared_ptr<HardwareSpec> s;
};
struct qc_topology {
  std::shared_ptr<Topology> t;
};
struct qc_dataset {
  std::shared_ptr<Dataset> d;
  // identity of this handle for the pass-1 -> pass-2 handoff (never reused,
  // unlike addresses)
  uint64_t uid = next_dataset_uid();
  static uint64_t next_dataset_uid() {
    static std::atomic<uint64_t> n{0};
    return ++n;
  }
};
struct qc_stats {
  CalibrationStats s;
};
#ifdef QUANTC_B200
struct qc_comm {
  std::unique_ptr<Communicator> c;
};
#endif
struct qc_evaluator {
  // CandidateEvaluator borrows graph/spec/dataset (reference search.hpp:130-132);
  // the handle keeps them alive.
  std::shared_ptr<Graph> g;
  std::shared_ptr<HardwareSpec> s;
  std::shared_ptr<Dataset> d;
  std::unique_ptr<CandidateEvaluator> ev;
};

namespace {

thread_local std::string g_last_error;
thread_local int64_t g_ovf[3] = {-1, -1, 0};

struct BufferTooSmall : std::runtime_error {
  BufferTooSmall() : std::runtime_error("caller buffer too small") {}
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return QC_OK;
  } catch (const BufferTooSmall& e) {
    g_last_error = e.what();
    return QC_ERR_BUFFER;
  } catch (const OverflowError& e) {
    g_last_error = e.what();
    g_ovf[0] = e.node;
    g_ovf[1] = e.flat_index;
    g_ovf[2] = e.value;
    return QC_ERR_OVERFLOW;
  } catch (const EvalError& e) {
    g_last_error = e.what();
    return QC_ERR_EVAL;
  } catch (const GraphError& e) {
    g_last_error = e.what();
    return QC_ERR_GRAPH;
  } catch (const SpecError& e) {
    g_last_error = e.what();
    return QC_ERR_SPEC;
  } catch (const TopologyError& e) {
    g_last_error = e.what();
    return QC_ERR_TOPOLOGY;
  } catch (const CalibrationError& e) {
    g_last_error = e.what();
    return QC_ERR_CALIBRATION;
  } catch (const SearchError& e) {
    g_last_error = e.what();
    return QC_ERR_SEARCH;
#ifdef QUANTC_B200
  } catch (const DeviceError& e) {
    g_last_error = e.what();
    return QC_ERR_CUDA;
#endif
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return QC_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return QC_ERR_INTERNAL;
  } catch (...) {
    g_last_error = "unknown exception";
    return QC_ERR_INTERNAL;
  }
}

int run(const std::function<void()>& f) {
  try {
    return guarded(f);
  } catch (...) {
    return QC_ERR_INTERNAL;
  }
}

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

DType dtype_of(int code) {
  if (code < QC_F32 || code > QC_I32) throw std::invalid_argument("bad dtype code");
  return DType(static_cast<DTypeKind>(code));
}
int code_of(DType d) { return static_cast<int>(d.kind); }

QParams from_pod(const qc_qparams& p) {
  QParams q;
  q.threshold = p.threshold;
  q.bit = p.bit;
  q.sign = p.sign;
  q.in_dtype = dtype_of(p.in_dtype);
  q.out_dtype = dtype_of(p.out_dtype);
  q.zero_point = p.zero_point;
  q.passthrough = p.passthrough != 0;
  if (p.acc_dtype != QC_NONE) q.acc_dtype = dtype_of(p.acc_dtype);
  q.acc_scale = p.acc_scale;
  return q;
}

qc_qparams to_pod(const QParams& q) {
  qc_qparams p{};
  p.threshold = q.threshold;
  p.bit = q.bit;
  p.sign = q.sign;
  p.in_dtype = code_of(q.in_dtype);
  p.out_dtype = code_of(q.out_dtype);
  p.zero_point = q.zero_point;
  p.passthrough = q.passthrough ? 1 : 0;
  p.acc_dtype = q.acc_dtype.has_value() ? code_of(*q.acc_dtype) : QC_NONE;
  p.acc_scale = q.acc_scale;
  return p;
}

SimBinding make_binding(const int64_t* nodes, const qc_qparams* params, size_t n) {
  SimBinding b;
  for (size_t i = 0; i < n; ++i) b[nodes[i]] = from_pod(params[i]);
  return b;
}

template <typename T, typename S>
void emit(const std::vector<S>& src, T* out, size_t cap, size_t* n) {
  if (n) *n = src.size();
  if (src.size() > cap || (!out && !src.empty())) {
    if (cap == 0 && !out) return;  // size query
    throw BufferTooSmall();
  }
  for (size_t i = 0; i < src.size(); ++i) out[i] = static_cast<T>(src[i]);
}

Tensor input_tensor(const float* input, const int64_t* shape, int ndim) {
  std::vector<int64_t> sh(shape, shape + ndim);
  int64_t n = shape_numel(sh);
  return Tensor::from_floats(sh, std::vector<float>(input, input + n));
}

FeedMap single_feed(const Graph& g, Tensor t) {
  if (g.inputs().size() != 1) throw EvalError("C-ABI eval supports single-input graphs");
  Sample s;
  s.inputs.push_back(std::move(t));
  return feed_for(g, s);
}

Json tensor_meta(const Tensor& t, int64_t offset) {
  return Json{{"dtype", t.dtype().name()}, {"shape", t.shape()}, {"offset", offset}};
}

std::string trace_to_json(const SearchResult& r) {
  Json recs = Json::array();
  for (const TraceRecord& t : r.trace.records) {
    recs.push_back(Json::array({t.iteration, t.bits, t.loss, t.accepted}));
  }
  return Json{{"header", r.trace.header}, {"records", recs}}.dump();
}

}  // namespace

extern "C" {

const char* qc_last_error(void) { return g_last_error.c_str(); }

void qc_last_overflow(int64_t* node, int64_t* flat_index, int64_t* value) {
  if (node) *node = g_ovf[0];
  if (flat_index) *flat_index = g_ovf[1];
  if (value) *value = g_ovf[2];
}

const char* qc_impl_name(void) {
#ifdef QUANTC_B200
  return "quantc-b200";
#else
  return "quantc-reference";
#endif
}

void qc_free(void* p) { std::free(p); }

// ---- graph ----------------------------------------------------------------

int qc_graph_from_json(const char* json, const void* blob, size_t blob_len, qc_graph** out) {
  return run([&] {
    Json doc = Json::parse(json);
    const auto* bytes = static_cast<const uint8_t*>(blob);
    std::vector<Node> nodes;
    for (const Json& jn : doc.at("nodes")) {
      Node n;
      n.id = jn.at("id").get<NodeId>();
      n.op = parse_op(jn.at("op").get<std::string>());
      if (jn.contains("attrs") && jn.at("attrs").is_object()) n.attrs = jn.at("attrs");
      if (jn.contains("payload")) {
        const Json& pl = jn.at("payload");
        DType dt = parse_dtype(pl.at("dtype").get<std::string>());
        auto shape = pl.at("shape").get<std::vector<int64_t>>();
        int64_t off = pl.at("offset").get<int64_t>();
        int64_t count = shape_numel(shape);
        if (off < 0 || static_cast<size_t>(off + count * 4) > blob_len) {
          throw std::invalid_argument("payload of node " + std::to_string(n.id) +
                                      " exceeds the blob");
        }
        if (dt.is_float()) {
          std::vector<float> v(static_cast<size_t>(count));
          std::memcpy(v.data(), bytes + off, v.size() * 4);
          n.payload = Tensor::from_floats(shape, std::move(v));
        } else {
          std::vector<int32_t> v(static_cast<size_t>(count));
          std::memcpy(v.data(), bytes + off, v.size() * 4);
          n.payload = Tensor::from_ints(dt, shape, std::move(v));
        }
      }
      nodes.push_back(std::move(n));
    }
    std::vector<Edge> edges;
    for (const Json& je : doc.at("edges")) {
      Edge e;
      e.src = PortRef{je.at("src")[0].get<NodeId>(), je.at("src")[1].get<int>()};
      e.dst = PortRef{je.at("dst")[0].get<NodeId>(), je.at("dst")[1].get<int>()};
      edges.push_back(e);
    }
    std::vector<NodeId> inputs = doc.at("inputs").get<std::vector<NodeId>>();
    std::vector<PortRef> outputs;
    for (const Json& jo : doc.at("outputs")) {
      outputs.push_back(PortRef{jo[0].get<NodeId>(), jo[1].get<int>()});
    }
    auto h = std::make_unique<qc_graph>();
    h->g = std::make_shared<Graph>(std::move(nodes), std::move(edges), std::move(inputs),
                                   std::move(outputs));
    *out = h.release();
  });
}

int qc_graph_to_json(const qc_graph* g, char** json_out) {
  return run([&] {
    Json nodes = Json::array();
    int64_t offset = 0;
    for (const Node& n : g->g->nodes()) {
      Json jn = {{"id", n.id}, {"op", op_name(n.op)}, {"attrs", n.attrs}};
      if (n.payload.has_value()) {
        jn["payload"] = tensor_meta(*n.payload, offset);
        offset += n.payload->numel() * 4;
      }
      nodes.push_back(jn);
    }
    Json edges = Json::array();
    for (const Edge& e : g->g->edges()) {
      edges.push_back({{"src", {e.src.node, e.src.port}}, {"dst", {e.dst.node, e.dst.port}}});
    }
    Json outs = Json::array();
    for (const PortRef& p : g->g->outputs()) outs.push_back({p.node, p.port});
    Json doc = {{"nodes", nodes}, {"edges", edges}, {"inputs", g->g->inputs()}, {"outputs", outs}};
    *json_out = dup_string(doc.dump());
  });
}

int qc_graph_blob(const qc_graph* g, void* out, size_t cap, size_t* n) {
  return run([&] {
    size_t total = 0;
    for (const Node& nd : g->g->nodes()) {
      if (nd.payload.has_value()) total += static_cast<size_t>(nd.payload->numel()) * 4;
    }
    *n = total;
    if (total > cap) throw BufferTooSmall();
    auto* dst = static_cast<uint8_t*>(out);
    for (const Node& nd : g->g->nodes()) {
      if (!nd.payload.has_value()) continue;
      const Tensor& t = *nd.payload;
      const void* src = t.dtype().is_float() ? static_cast<const void*>(t.floats().data())
                                             : static_cast<const void*>(t.ints().data());
      std::memcpy(dst, src, static_cast<size_t>(t.numel()) * 4);
      dst += static_cast<size_t>(t.numel()) * 4;
    }
  });
}

void qc_graph_free(qc_graph* g) { delete g; }

int qc_graph_num_nodes(const qc_graph* g, size_t* n) {
  return run([&] { *n = g->g->nodes().size(); });
}

int qc_validate_graph(const qc_graph* g, char** report_json) {
  return run([&] {
    Json rep = Json::array();
    for (const Violation& v : validate_graph(*g->g)) {
      rep.push_back({{"node", v.node}, {"message", v.message}});
    }
    *report_json = dup_string(rep.dump());
  });
}

int qc_traversal_order(const qc_graph* g, int64_t* out, size_t cap, size_t* n) {
  return run([&] { emit(traversal_order(*g->g), out, cap, n); });
}

int qc_edge_order(const qc_graph* g, int64_t* out, size_t cap, size_t* n_edges) {
  return run([&] {
    std::vector<int64_t> flat;
    for (const Edge& e : edge_order(*g->g)) {
      flat.insert(flat.end(), {e.src.node, e.src.port, e.dst.node, e.dst.port});
    }
    size_t n4 = 0;
    emit(flat, out, cap, &n4);
    if (n_edges) *n_edges = n4 / 4;
  });
}

// ---- files (quantc_files.h; B200 library only: the reference declares
// serialize.hpp without implementing it) ----------------------------------
#ifdef QUANTC_B200

int qc_graph_save(const qc_graph* g, const char* json_path) {
  return run([&] { save_graph(*g->g, json_path); });
}

int qc_graph_load(const char* json_path, qc_graph** out) {
  return run([&] { *out = new qc_graph{std::make_shared<Graph>(load_graph(json_path))}; });
}

int qc_stats_save(const qc_stats* s, const char* path) {
  return run([&] { save_stats(s->s, path); });
}

int qc_stats_load(const char* path, qc_stats** out) {
  return run([&] {
    auto h = std::make_unique<qc_stats>();
    h->s = load_stats(path);
    *out = h.release();
  });
}

int qc_fingerprint_graph(const qc_graph* g, uint64_t* out) {
  return run([&] { *out = fingerprint_graph(*g->g); });
}

int qc_fnv1a64(const void* data, size_t size, uint64_t seed, uint64_t* out) {
  return run([&] { *out = fnv1a64(data, size, seed); });
}

int qc_fixtures_write_all(const char* dir) {
  return run([&] { fixtures::write_all(dir); });
}

int qc_fixtures_verify_committed(const char* dir) {
  return run([&] { fixtures::verify_committed(dir); });
}
#endif  // QUANTC_B200

// ---- hwspec ---------------------------------------------------------------

int qc_spec_parse(const char* text, qc_spec** out) {
  return run([&] {
    auto h = std::make_unique<qc_spec>();
    h->s = std::make_shared<HardwareSpec>(parse_spec(text));
    *out = h.release();
  });
}

void qc_spec_free(qc_spec* s) { delete s; }

int qc_spec_serialize(const qc_spec* s, char** text) {
  return run([&] { *text = dup_string(serialize_spec(*s->s)); });
}

int qc_classify_op(const qc_spec* s, const char* op, int* cls) {
  return run([&] {
    OpClass c = classify_op(*s->s, parse_op(op));
    *cls = c == OpClass::kFloatOnly ? 0 : c == OpClass::kIntegerOnly ? 1 : 2;
  });
}

int qc_candidate_dtypes(const qc_spec* s, const char* op, int port, int* out, size_t cap,
                        size_t* n) {
  return run([&] {
    std::vector<int> codes;
    for (DType d : candidate_dtypes(*s->s, parse_op(op), port)) codes.push_back(code_of(d));
    emit(codes, out, cap, n);
  });
}

int qc_match_signature(const qc_spec* s, const char* op, const int* bits, const int* signs,
                       size_t n, int* found, int* in_dtypes, int* out_dtype) {
  return run([&] {
    std::vector<Signature> sigs = s->s->signatures(parse_op(op));
    const Signature* sig = match_signature(sigs, std::vector<int>(bits, bits + n),
                                           std::vector<int>(signs, signs + n));
    *found = sig ? 1 : 0;
    if (sig) {
      for (size_t i = 0; i < sig->in_dtypes.size(); ++i) in_dtypes[i] = code_of(sig->in_dtypes[i]);
      *out_dtype = code_of(sig->out_dtype);
    }
  });
}

// ---- topology -------------------------------------------------------------

int qc_generate_topology(const qc_graph* g, const qc_spec* s, qc_topology** out) {
  return run([&] {
    auto h = std::make_unique<qc_topology>();
    h->t = std::make_shared<Topology>(generate_topology(*g->g, *s->s));
    *out = h.release();
  });
}

void qc_topology_free(qc_topology* t) { delete t; }

int qc_dump_topology(const qc_graph* g, const qc_topology* t, char** json) {
  return run([&] { *json = dup_string(dump_topology(*g->g, *t->t)); });
}

int qc_topology_qv(const qc_topology* t, int64_t* out, size_t cap, size_t* n) {
  return run([&] {
    std::vector<int64_t> v(t->t->qv.begin(), t->t->qv.end());
    emit(v, out, cap, n);
  });
}

int qc_insert_simulated_quantize(const qc_graph* g, const qc_topology* t, qc_graph** out) {
  return run([&] {
    auto h = std::make_unique<qc_graph>();
    h->g = std::make_shared<Graph>(insert_simulated_quantize(*g->g, *t->t));
    *out = h.release();
  });
}

int qc_searchable_edge_indices(const qc_topology* t, int* out, size_t cap, size_t* n) {
  return run([&] { emit(searchable_edge_indices(*t->t), out, cap, n); });
}

int qc_simulated_edge_indices(const qc_graph* g, const qc_topology* t, int* out, size_t cap,
                              size_t* n) {
  return run([&] { emit(simulated_edge_indices(*g->g, *t->t), out, cap, n); });
}

// ---- dataset --------------------------------------------------------------

int qc_dataset_create(const float* data, int64_t n_samples, const int64_t* sample_shape,
                      int ndim, const int64_t* labels, qc_dataset** out) {
  return run([&] {
    std::vector<int64_t> sh(sample_shape, sample_shape + ndim);
    int64_t per = shape_numel(sh);
#ifdef QUANTC_B200
    // B200: a contiguous page-locked mirror of the samples (one DMA per
    // upload), else the samples' own storage page-locked (device.hpp)
    const size_t total_bytes = static_cast<size_t>(n_samples) * static_cast<size_t>(per) * 4;
    void* mirror = device::alloc_pinned(total_bytes);
    if (mirror) std::memcpy(mirror, data, total_bytes);
    auto ds = std::shared_ptr<Dataset>(new Dataset, [mirror](Dataset* p) {
      if (mirror) {
        device::clear_dataset_mirror(p);
        device::free_pinned(mirror);
      }
      for (const Sample& s : *p) {
        for (const Tensor& t : s.inputs) {
          if (t.dtype().is_float() && t.numel() > 0) device::unpin_host(t.floats().data());
        }
      }
      delete p;
    });
#else
    auto ds = std::make_shared<Dataset>();
#endif
    ds->reserve(static_cast<size_t>(n_samples));
    for (int64_t i = 0; i < n_samples; ++i) {
      Sample s;
      s.inputs.push_back(Tensor::from_floats(
          sh, std::vector<float>(data + i * per, data + (i + 1) * per)));
      if (labels) s.label = labels[i];
      ds->push_back(std::move(s));
    }
#ifdef QUANTC_B200
    if (mirror) {
      device::set_dataset_mirror(ds.get(), mirror, static_cast<size_t>(per) * 4, n_samples);
    } else {
      for (const Sample& s : *ds) {
        const Tensor& t = s.inputs[0];
        if (t.numel() > 0) device::pin_host(t.floats().data(), static_cast<size_t>(t.numel()) * 4);
      }
    }
#endif
    auto h = std::make_unique<qc_dataset>();
    h->d = std::move(ds);
    *out = h.release();
  });
}

#ifdef QUANTC_B200
// dataset manifest (serialize.hpp load_dataset; quantc_files.h): single-input
// samples of one shape, rebuilt through qc_dataset_create (page-locked mirror)
int qc_dataset_load(const char* manifest_path, qc_dataset** out, int64_t* n_samples) {
  Dataset d;
  int rc = run([&] {
    d = load_dataset(manifest_path);
    if (d.empty()) throw IoError(std::string("empty dataset: ") + manifest_path);
    for (const Sample& s : d) {
      if (s.inputs.size() != 1 || s.inputs[0].shape() != d[0].inputs[0].shape() || !s.inputs[0].dtype().is_float()) {
        throw IoError(std::string("qc_dataset_load: samples must share one fp32 input shape: ") + manifest_path);
      }
    }
  });
  if (rc != 0) return rc;
  const auto& sh = d[0].inputs[0].shape();
  const size_t per = static_cast<size_t>(d[0].inputs[0].numel());
  std::vector<float> flat(per * d.size());
  std::vector<int64_t> labels(d.size(), -1);
  bool any_label = false;
  for (size_t i = 0; i < d.size(); ++i) {
    const auto v = d[i].inputs[0].floats();
    std::copy(v.begin(), v.end(), flat.begin() + static_cast<std::ptrdiff_t>(i * per));
    if (d[i].label) {
      labels[i] = *d[i].label;
      any_label = true;
    }
  }
  if (n_samples) *n_samples = static_cast<int64_t>(d.size());
  return qc_dataset_create(flat.data(), static_cast<int64_t>(d.size()), sh.data(),
                           static_cast<int>(sh.size()), any_label ? labels.data() : nullptr, out);
}
#endif  // QUANTC_B200

void qc_dataset_free(qc_dataset* d) { delete d; }

// ---- simulate -------------------------------------------------------------

int qc_compute_scale(double threshold, int bit, int sign, double* out) {
  return run([&] { *out = compute_scale(threshold, bit, sign); });
}

int qc_quant_bounds(int bit, int sign, int64_t* qmin, int64_t* qmax) {
  return run([&] {
    QuantBounds b = quant_bounds(bit, sign);
    *qmin = b.qmin;
    *qmax = b.qmax;
  });
}

int qc_simulated_quantize_value(float x, const qc_qparams* p, float* out) {
  return run([&] { *out = simulated_quantize_value(x, from_pod(*p)); });
}

int qc_simulated_quantize(const float* x, int64_t n, const qc_qparams* p, float* out) {
  return run([&] {
    Tensor t = Tensor::from_floats({n}, std::vector<float>(x, x + n));
    Tensor r = simulated_quantize(t, from_pod(*p));
    auto f = r.floats();
    std::memcpy(out, f.data(), static_cast<size_t>(n) * sizeof(float));
  });
}

int qc_asymmetric_zero_point(double min_value, double range_threshold, int bit, int64_t* out) {
  return run([&] { *out = asymmetric_zero_point(min_value, range_threshold, bit); });
}

int qc_noop_params(qc_qparams* out) {
  return run([&] { *out = to_pod(noop_params()); });
}

// ---- calibration ----------------------------------------------------------

int qc_collect_stats(const qc_graph* g, const qc_dataset* d, int bins, const int* edges,
                     size_t n_edges, int workers, qc_stats** out) {
  return run([&] {
    std::vector<int> e(edges, edges + n_edges);
    auto h = std::make_unique<qc_stats>();
    h->s = collect_stats(*g->g, *d->d, bins, e, workers);
    *out = h.release();
  });
}

int qc_stats_create(qc_stats** out) {
  return run([&] { *out = new qc_stats(); });
}

int qc_stats_set_edge(qc_stats* s, int edge, double min, double max, double absmax,
                      int64_t sample_count, const int64_t* counts, size_t bins) {
  return run([&] {
    EdgeStats e;
    e.min = min;
    e.max = max;
    e.absmax = absmax;
    e.sample_count = sample_count;
    e.counts.assign(counts, counts + bins);
    s->s.per_edge[edge] = std::move(e);
  });
}

void qc_stats_free(qc_stats* s) { delete s; }

int qc_stats_edges(const qc_stats* s, int* out, size_t cap, size_t* n) {
  return run([&] {
    std::vector<int> v;
    for (const auto& kv : s->s.per_edge) v.push_back(kv.first);
    emit(v, out, cap, n);
  });
}

int qc_stats_get(const qc_stats* s, int edge, double* min, double* max, double* absmax,
                 int64_t* sample_count, int64_t* counts, size_t cap, size_t* bins) {
  return run([&] {
    auto it = s->s.per_edge.find(edge);
    if (it == s->s.per_edge.end()) throw std::invalid_argument("no stats for edge");
    const EdgeStats& e = it->second;
    if (min) *min = e.min;
    if (max) *max = e.max;
    if (absmax) *absmax = e.absmax;
    if (sample_count) *sample_count = e.sample_count;
    emit(e.counts, counts, cap, bins);
  });
}

int qc_estimate_thresholds(const qc_stats* s, int method, double quantile, int kl_bits,
                           int pow2, int* edges_out, double* thresholds_out, size_t cap,
                           size_t* n) {
  return run([&] {
    ThresholdConfig cfg;
    cfg.method = method == 0   ? ThresholdMethod::kMax
                 : method == 1 ? ThresholdMethod::kQuantile
                               : ThresholdMethod::kKl;
    if (method < 0 || method > 2) throw std::invalid_argument("bad threshold method");
    cfg.quantile = quantile;
    cfg.kl_bits = kl_bits;
    cfg.pow2 = pow2 != 0;
    auto res = estimate_thresholds(s->s, cfg);
    std::vector<int> ks;
    std::vector<double> vs;
    for (const auto& kv : res) {
      ks.push_back(kv.first);
      vs.push_back(kv.second);
    }
    emit(ks, edges_out, cap, n);
    emit(vs, thresholds_out, cap, n);
  });
}

namespace {
EdgeStats edge_from(const int64_t* counts, size_t bins, double absmax) {
  EdgeStats e;
  e.absmax = absmax;
  e.max = absmax;
  e.min = -absmax;
  e.counts.assign(counts, counts + bins);
  e.sample_count = 1;
  return e;
}
}  // namespace

int qc_threshold_max(double absmax, double* out) {
  return run([&] {
    EdgeStats e;
    e.absmax = absmax;
    *out = threshold_max(e);
  });
}

int qc_threshold_quantile(const int64_t* counts, size_t bins, double absmax, double q,
                          double* out) {
  return run([&] { *out = threshold_quantile(edge_from(counts, bins, absmax), q); });
}

int qc_threshold_kl(const int64_t* counts, size_t bins, double absmax, int target_bit,
                    double* out) {
  return run([&] { *out = threshold_kl(edge_from(counts, bins, absmax), target_bit); });
}

int qc_round_pow2(double threshold, double* out) {
  return run([&] { *out = round_pow2(threshold); });
}

// ---- interpreter ----------------------------------------------------------

int qc_eval_fp32(const qc_graph* g, const float* input, const int64_t* shape, int ndim,
                 const int64_t* bind_nodes, const qc_qparams* bind_params, size_t n_bind,
                 float* out, size_t cap, size_t* n_out, int64_t* out_shape, int* out_ndim) {
  return run([&] {
    SimBinding b = make_binding(bind_nodes, bind_params, n_bind);
#ifdef QUANTC_B200
    // the caller's buffer is uploaded directly (no Tensor / FeedMap copies)
    std::vector<Tensor> outs = engine::eval_fp32_host(*g->g, input, std::vector<int64_t>(shape, shape + ndim),
                                                      n_bind ? &b : nullptr);
#else
    FeedMap feed = single_feed(*g->g, input_tensor(input, shape, ndim));
    std::vector<Tensor> outs = eval_fp32(*g->g, feed, n_bind ? &b : nullptr);
#endif
    if (outs.empty()) throw EvalError("graph has no outputs");
    const Tensor& t = outs[0];
    if (out_ndim) *out_ndim = static_cast<int>(t.shape().size());
    if (out_shape) {
      for (size_t i = 0; i < t.shape().size(); ++i) out_shape[i] = t.shape()[i];
    }
    auto f = t.floats();
    emit(std::vector<float>(f.begin(), f.end()), out, cap, n_out);
  });
}

int qc_eval_fp32_values(const qc_graph* g, const float* input, const int64_t* shape, int ndim,
                        const int64_t* nodes, size_t n_nodes, float* out, size_t cap,
                        size_t* n_out) {
  return run([&] {
    FeedMap feed = single_feed(*g->g, input_tensor(input, shape, ndim));
    auto values = eval_fp32_values(*g->g, feed);
    std::vector<float> flat;
    for (size_t i = 0; i < n_nodes; ++i) {
      auto f = values.at(nodes[i]).floats();
      flat.insert(flat.end(), f.begin(), f.end());
    }
    emit(flat, out, cap, n_out);
  });
}

int qc_eval_int(const qc_graph* g, const float* input, const int64_t* shape, int ndim,
                int mode, int32_t* out, size_t cap, size_t* n_out, int* out_dtype) {
  return run([&] {
#ifdef QUANTC_B200
    auto outs = engine::eval_int_host(*g->g, input, std::vector<int64_t>(shape, shape + ndim),
                                      mode ? OverflowMode::kTrap : OverflowMode::kSaturate);
#else
    FeedMap feed = single_feed(*g->g, input_tensor(input, shape, ndim));
    auto outs = eval_int(*g->g, feed, mode ? OverflowMode::kTrap : OverflowMode::kSaturate);
#endif
    if (outs.empty()) throw EvalError("graph has no outputs");
    const Tensor& t = outs[0];
    *out_dtype = code_of(t.dtype());
    std::vector<int32_t> raw(static_cast<size_t>(t.numel()));
    if (t.dtype().is_float()) {
      std::memcpy(raw.data(), t.floats().data(), raw.size() * 4);
    } else {
      std::memcpy(raw.data(), t.ints().data(), raw.size() * 4);
    }
    emit(raw, out, cap, n_out);
  });
}

int qc_predict_top1(const qc_graph* g, const qc_dataset* d, int workers,
                    const int64_t* bind_nodes, const qc_qparams* bind_params, size_t n_bind,
                    int64_t* out, size_t cap, size_t* n) {
  return run([&] {
    SimBinding b = make_binding(bind_nodes, bind_params, n_bind);
    emit(predict_top1(*g->g, *d->d, workers, n_bind ? &b : nullptr), out, cap, n);
  });
}

// ---- search ---------------------------------------------------------------

int qc_evaluator_create(const qc_graph* sim_g, const qc_spec* spec, const qc_topology* t,
                        const int* thr_edges, const double* thr_values, size_t n_thr,
                        const qc_stats* stats, const qc_dataset* calib, int min_bit,
                        int workers, qc_evaluator** out) {
  return run([&] {
    std::map<int, double> thr;
    for (size_t i = 0; i < n_thr; ++i) thr[thr_edges[i]] = thr_values[i];
    auto h = std::make_unique<qc_evaluator>();
    h->g = sim_g->g;
    h->s = spec->s;
    h->d = calib->d;
    h->ev = std::make_unique<CandidateEvaluator>(*h->g, *h->s, *t->t, thr, stats->s, *h->d,
                                                 min_bit, workers);
    *out = h.release();
  });
}

void qc_evaluator_free(qc_evaluator* e) { delete e; }

int qc_evaluator_space(const qc_evaluator* e, int* edges, int* lo, int* hi, size_t cap,
                       size_t* n) {
  return run([&] {
    std::vector<int> ee, ll, hh;
    for (const BitRange& r : e->ev->space().ranges) {
      ee.push_back(r.edge_index);
      ll.push_back(r.lo);
      hh.push_back(r.hi);
    }
    emit(ee, edges, cap, n);
    emit(ll, lo, cap, n);
    emit(hh, hi, cap, n);
  });
}

int qc_evaluator_refs(const qc_evaluator* e, int64_t* out, size_t cap, size_t* n) {
  return run([&] { emit(e->ev->reference_predictions(), out, cap, n); });
}

int qc_evaluator_bind(const qc_evaluator* e, const int* cand, size_t n_slots,
                      int64_t* nodes_out, qc_qparams* params_out, size_t cap, size_t* n) {
  return run([&] {
    SimBinding b = e->ev->bind(Candidate(cand, cand + n_slots));
    std::vector<int64_t> ids;
    std::vector<qc_qparams> ps;
    for (const auto& kv : b) {
      ids.push_back(kv.first);
      ps.push_back(to_pod(kv.second));
    }
    emit(ids, nodes_out, cap, n);
    if (n) *n = ps.size();
    if (ps.size() > cap) throw BufferTooSmall();
    for (size_t i = 0; i < ps.size(); ++i) params_out[i] = ps[i];
  });
}

int qc_evaluator_loss(const qc_evaluator* e, const int* cand, size_t n_slots, double* out) {
  return run([&] { *out = e->ev->loss(Candidate(cand, cand + n_slots)); });
}

int qc_evaluator_losses(const qc_evaluator* e, const int* cands, size_t n_cands,
                        size_t n_slots, double* out) {
  return run([&] {
    std::vector<Candidate> cs;
    for (size_t i = 0; i < n_cands; ++i) {
      cs.emplace_back(cands + i * n_slots, cands + (i + 1) * n_slots);
    }
    std::vector<double> ls = e->ev->losses(std::span<const Candidate>(cs.data(), cs.size()));
    for (size_t i = 0; i < ls.size(); ++i) out[i] = ls[i];
  });
}

int qc_evaluator_strategy(const qc_evaluator* e, const int* cand, size_t n_slots, char** json) {
  return run([&] {
    Strategy st = e->ev->strategy_for(Candidate(cand, cand + n_slots));
    Json doc = Json::object();
    for (const auto& kv : st.edges) {
      const EdgeDecision& d = kv.second;
      doc[std::to_string(kv.first)] = {{"bit", d.bit},
                                       {"threshold", d.threshold},
                                       {"sign", d.sign},
                                       {"zero_point", d.zero_point},
                                       {"storage_dtype", d.storage_dtype.name()}};
    }
    *json = dup_string(doc.dump());
  });
}

#ifdef QUANTC_B200
int qc_requantize_params(double s_in, double s_out, int32_t* multiplier, int* shift) {
  return run([&] {
    const RequantParams r = requantize_params(s_in, s_out);
    *multiplier = r.multiplier;
    *shift = r.shift;
  });
}

int qc_choose_storage_dtype(int bit, const char* candidates_csv, int sign, char* out,
                            size_t cap) {
  return run([&] {
    std::vector<DType> cands;
    std::string all(candidates_csv), tok;
    std::stringstream ss(all);
    while (std::getline(ss, tok, ',')) {
      if (!tok.empty()) cands.push_back(parse_dtype(tok));
    }
    const std::string name = choose_storage_dtype(bit, cands, sign).name();
    if (name.size() + 1 > cap) throw BufferTooSmall();
    std::memcpy(out, name.c_str(), name.size() + 1);
  });
}

int qc_rewrite_clip(double min_f, double max_f, double s_out, int64_t zero_point,
                    const char* storage, int64_t* q_min, int64_t* q_max) {
  return run([&] {
    const auto [lo, hi] = rewrite_clip(min_f, max_f, s_out, zero_point, parse_dtype(storage));
    *q_min = lo;
    *q_max = hi;
  });
}

int qc_realize(const qc_graph* sim_g, const char* strategy_json, const qc_spec* spec,
               qc_graph** out) {
  return run([&] {
    Strategy st;
    const Json doc = Json::parse(strategy_json);  // items() must not outlive it
    for (const auto& kv : doc.items()) {
      EdgeDecision d;
      d.bit = kv.value().at("bit").get<int>();
      d.threshold = kv.value().at("threshold").get<double>();
      d.sign = kv.value().at("sign").get<int>();
      d.zero_point = kv.value().at("zero_point").get<int64_t>();
      d.storage_dtype = parse_dtype(kv.value().at("storage_dtype").get<std::string>());
      st.edges[std::stoi(kv.key())] = d;
    }
    auto h = std::make_unique<qc_graph>();
    h->g = std::make_shared<Graph>(realize(*sim_g->g, st, *spec->s));
    *out = h.release();
  });
}

int qc_collect_extrema(const qc_graph* g, const qc_dataset* d, const int* edges, size_t n,
                       double* mins, double* maxs) {
  return run([&] {
    std::vector<double> lo, hi;
    collect_extrema(*g->g, *d->d, std::vector<int>(edges, edges + n), &lo, &hi, d->uid);
    std::copy(lo.begin(), lo.end(), mins);
    std::copy(hi.begin(), hi.end(), maxs);
  });
}

int qc_collect_histograms(const qc_graph* g, const qc_dataset* d, const int* edges, size_t n,
                          const double* absmax, int bins, int64_t* counts) {
  return run([&] {
    std::vector<int64_t> c;
    collect_histograms(*g->g, *d->d, std::vector<int>(edges, edges + n),
                       std::vector<double>(absmax, absmax + n), bins, &c, d->uid);
    std::copy(c.begin(), c.end(), counts);
  });
}

int qc_predict_scores(const qc_graph* g, const qc_dataset* d, const int64_t* bind_nodes,
                      const qc_qparams* bind_params, size_t n_bind, float* out, size_t cap,
                      size_t* n_out, int64_t* per_sample) {
  return run([&] {
    SimBinding b = make_binding(bind_nodes, bind_params, n_bind);
    emit(predict_scores(*g->g, *d->d, n_bind ? &b : nullptr, per_sample), out, cap, n_out);
  });
}

int qc_fused_status(const qc_graph* g, const int64_t* bind_nodes, const qc_qparams* bind_params,
                    size_t n_bind, char** why) {
  return run([&] {
    SimBinding b = make_binding(bind_nodes, bind_params, n_bind);
    *why = dup_string(fused_status(*g->g, n_bind ? &b : nullptr));
  });
}

int qc_evaluator_scores(const qc_evaluator* e, const int* cands, size_t n_cands, size_t n_slots,
                        int group, float* out, size_t cap, size_t* n_out, int64_t* per_sample) {
  return run([&] {
    std::vector<Candidate> cs;
    for (size_t i = 0; i < n_cands; ++i) {
      cs.emplace_back(cands + i * n_slots, cands + (i + 1) * n_slots);
    }
    emit(e->ev->scores(std::span<const Candidate>(cs.data(), cs.size()), group, per_sample), out,
         cap, n_out);
  });
}

int qc_comm_local(qc_comm** out) {
  return run([&] { *out = new qc_comm{make_local_communicator()}; });
}

int qc_comm_nccl_unique_id(char id[128]) {
  return run([&] {
    const NcclId u = nccl_unique_id();
    std::memcpy(id, u.data(), u.size());
  });
}

int qc_comm_nccl(int rank, int world, const char id[128], qc_comm** out) {
  return run([&] {
    NcclId u;
    std::memcpy(u.data(), id, u.size());
    *out = new qc_comm{make_nccl_communicator(rank, world, u)};
  });
}

int qc_comm_callbacks(int rank, int world, qc_comm_sum_i64_fn sum_i64, qc_comm_f64_fn minmax_f64,
                      qc_comm_gather_f64_fn gather_f64, void* user, qc_comm** out) {
  return run([&] {
    CommHooks h;
    h.rank = rank;
    h.size = world;
    h.user = user;
    h.allreduce_sum_i64 = sum_i64;
    h.allreduce_f64 = minmax_f64;
    h.allgather_f64 = gather_f64;
    *out = new qc_comm{make_callback_communicator(h)};
  });
}

void qc_comm_free(qc_comm* c) { delete c; }

int qc_collect_stats_dist(const qc_graph* g, const qc_dataset* d, qc_comm* comm, int bins,
                          const int* edges, size_t n_edges, qc_stats** out) {
  return run([&] {
    auto h = std::make_unique<qc_stats>();
    h->s = collect_stats(*g->g, *d->d, *comm->c, bins,
                         std::vector<int>(edges, edges + n_edges));
    *out = h.release();
  });
}

int qc_search_batched(int method, const int* edges, const int* lo, const int* hi, size_t n_slots,
                      qc_batch_loss_fn fn, void* user, const qc_evaluator* ev, qc_comm* comm,
                      int loss_mode, const qc_search_params* p, int width, int* best,
                      double* best_loss, int64_t* evaluations, char** trace_json,
                      int64_t* spec_stats) {
  return run([&] {
    SearchSpace space;
    for (size_t i = 0; i < n_slots; ++i) space.ranges.push_back(BitRange{edges[i], lo[i], hi[i]});
    BatchLossFn losses;
    if (fn) {
      losses = [fn, user, n_slots](std::span<const Candidate> cs) {
        std::vector<int> flat;
        flat.reserve(cs.size() * n_slots);
        for (const Candidate& c : cs) flat.insert(flat.end(), c.begin(), c.end());
        std::vector<double> v(cs.size());
        if (fn(flat.data(), cs.size(), n_slots, user, v.data()) != 0) {
          throw SearchError("loss callback failed");
        }
        return v;
      };
      if (loss_mode == QC_LOSS_CANDIDATES) {
        if (!comm) throw std::invalid_argument("sharded losses need a communicator");
        losses = shard_candidates(std::move(losses), *comm->c);
      } else if (loss_mode != QC_LOSS_LOCAL) {
        throw std::invalid_argument("a batch callback supports local or candidate sharding");
      }
    } else if (ev) {
      const CandidateEvaluator& E = *ev->ev;
      if (loss_mode == QC_LOSS_SAMPLES || loss_mode == QC_LOSS_CANDIDATES) {
        if (!comm) throw std::invalid_argument("sharded losses need a communicator");
        losses = loss_mode == QC_LOSS_SAMPLES ? sample_sharded_losses(E, *comm->c)
                                              : candidate_sharded_losses(E, *comm->c);
      } else {
        losses = E.batch_loss();
      }
    } else {
      throw std::invalid_argument("qc_search_batched needs a loss callback or an evaluator");
    }
    SpeculationStats st;
    SearchResult r;
    switch (method) {
      case QC_SEARCH_GREEDY:
        r = greedy_search_batched(space, losses, p->rounds, p->tol, width, &st);
        break;
      case QC_SEARCH_ANNEAL:
        r = anneal_search_batched(space, losses, p->steps, p->t0, p->decay, p->seed, width, &st);
        break;
      case QC_SEARCH_RANDOM:
        r = random_search_batched(space, losses, p->n, p->seed, width, &st);
        break;
      case QC_SEARCH_EXHAUSTIVE:
        r = exhaustive_search_batched(space, losses, p->cap, width, &st);
        break;
      default:
        throw std::invalid_argument("unknown search method");
    }
    for (size_t i = 0; i < r.best.size(); ++i) best[i] = r.best[i];
    *best_loss = r.best_loss;
    *evaluations = r.evaluations;
    if (trace_json) *trace_json = dup_string(trace_to_json(r));
    if (spec_stats) {
      spec_stats[0] = st.batches;
      spec_stats[1] = st.evaluated;
      spec_stats[2] = st.committed;
    }
  });
}

int qc_evaluator_agreement(const qc_evaluator* e, const int* cands, size_t n_cands,
                           size_t n_slots, int64_t* counts) {
  return run([&] {
    std::vector<Candidate> cs;
    for (size_t i = 0; i < n_cands; ++i) {
      cs.emplace_back(cands + i * n_slots, cands + (i + 1) * n_slots);
    }
    auto v = e->ev->agreement_counts(std::span<const Candidate>(cs.data(), cs.size()));
    for (size_t i = 0; i < v.size(); ++i) counts[i] = v[i];
  });
}
#endif

int qc_evaluator_evaluations(const qc_evaluator* e, int64_t* out) {
  return run([&] { *out = e->ev->evaluations(); });
}

int qc_search(int method, const int* edges, const int* lo, const int* hi, size_t n_slots,
              qc_loss_fn fn, void* user, const qc_evaluator* ev, const qc_search_params* p,
              int* best, double* best_loss, int64_t* evaluations, char** trace_json) {
  return run([&] {
    SearchSpace space;
    for (size_t i = 0; i < n_slots; ++i) {
      BitRange r;
      r.edge_index = edges[i];
      r.lo = lo[i];
      r.hi = hi[i];
      space.ranges.push_back(r);
    }
    LossFn loss;
    if (fn) {
      loss = [fn, user](const Candidate& c) {
        double v = 0.0;
        if (fn(c.data(), c.size(), user, &v) != 0) {
          throw SearchError("loss callback failed");
        }
        return v;
      };
    } else if (ev) {
      loss = [ev](const Candidate& c) { return ev->ev->loss(c); };
    } else {
      throw std::invalid_argument("qc_search needs a loss callback or an evaluator");
    }
    SearchResult r;
    switch (method) {
      case QC_SEARCH_GREEDY:
        r = greedy_search(space, loss, p->rounds, p->tol);
        break;
      case QC_SEARCH_ANNEAL:
        r = anneal_search(space, loss, p->steps, p->t0, p->decay, p->seed);
        break;
      case QC_SEARCH_RANDOM:
        r = random_search(space, loss, p->n, p->seed);
        break;
      case QC_SEARCH_EXHAUSTIVE:
        r = exhaustive_search(space, loss, p->cap);
        break;
      default:
        throw std::invalid_argument("unknown search method");
    }
    for (size_t i = 0; i < r.best.size(); ++i) best[i] = r.best[i];
    *best_loss = r.best_loss;
    *evaluations = r.evaluations;
    if (trace_json) *trace_json = dup_string(trace_to_json(r));
  });
}

int qc_space_size(const int* lo, const int* hi, size_t n_slots, char** decimal) {
  return run([&] {
    SearchSpace space;
    for (size_t i = 0; i < n_slots; ++i) {
      BitRange r;
      r.lo = lo[i];
      r.hi = hi[i];
      space.ranges.push_back(r);
    }
    *decimal = dup_string(space_size(space).str());
  });
}

}  // extern "C"
