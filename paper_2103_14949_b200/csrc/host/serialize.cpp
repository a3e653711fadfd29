// serialize.cpp — file formats of quantc/serialize.hpp (SPEC.md:102, :382,
// :583).  Host-only; no device code.
#include "quantc/serialize.hpp"

#include <cstring>
#include <fstream>
#include <map>
#include <sstream>

namespace quantc {

namespace {

namespace fs = std::filesystem;

std::string read_file(const fs::path& p) {
  std::ifstream f(p, std::ios::binary);
  if (!f) throw IoError("cannot open " + p.string());
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

void write_file(const fs::path& p, const std::string& bytes) {
  std::ofstream f(p, std::ios::binary | std::ios::trunc);
  if (!f) throw IoError("cannot write " + p.string());
  f.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
  if (!f) throw IoError("write failed: " + p.string());
}

Json parse_json(const fs::path& p) {
  try {
    return Json::parse(read_file(p));
  } catch (const Json::exception& e) {
    throw IoError("malformed JSON in " + p.string() + ": " + e.what());
  }
}

// element width in the sidecar: float32 / int32 4 bytes, int16 2, (u)int8 1
size_t elem_bytes(DType dt) {
  if (dt.is_float()) return 4;
  const int w = dt.width();
  return w <= 8 ? 1 : (w <= 16 ? 2 : 4);
}

// append t's elements little-endian at their natural width; returns offset
int64_t append_tensor(const Tensor& t, std::string* out) {
  const int64_t off = static_cast<int64_t>(out->size());
  const size_t eb = elem_bytes(t.dtype());
  if (t.dtype().is_float()) {
    auto v = t.floats();
    out->append(reinterpret_cast<const char*>(v.data()), v.size() * 4);  // host is little-endian
  } else {
    auto v = t.ints();
    for (int32_t x : v) {
      const uint32_t u = static_cast<uint32_t>(x);
      for (size_t b = 0; b < eb; ++b) out->push_back(static_cast<char>((u >> (8 * b)) & 0xFF));
    }
  }
  return off;
}

Tensor decode_tensor(const std::string& bytes, int64_t off, DType dt,
                     const std::vector<int64_t>& shape, const std::string& what) {
  const int64_t n = shape_numel(shape);
  const size_t eb = elem_bytes(dt);
  if (off < 0 || static_cast<size_t>(off) + static_cast<size_t>(n) * eb > bytes.size()) {
    throw IoError("tensor ref " + what + " exceeds its sidecar");
  }
  const auto* p = reinterpret_cast<const uint8_t*>(bytes.data()) + off;
  if (dt.is_float()) {
    std::vector<float> v(static_cast<size_t>(n));
    std::memcpy(v.data(), p, v.size() * 4);
    return Tensor::from_floats(shape, std::move(v));
  }
  std::vector<int32_t> v(static_cast<size_t>(n));
  const bool is_signed = dt.is_signed();
  for (int64_t i = 0; i < n; ++i) {
    uint32_t u = 0;
    for (size_t b = 0; b < eb; ++b) u |= static_cast<uint32_t>(p[i * eb + b]) << (8 * b);
    int32_t x = static_cast<int32_t>(u);
    if (is_signed && eb < 4) {  // sign-extend
      const int sh = static_cast<int>(32 - 8 * eb);
      x = static_cast<int32_t>(u << sh) >> sh;
    }
    v[static_cast<size_t>(i)] = x;
  }
  return Tensor::from_ints(dt, shape, std::move(v));
}

Json tensor_ref(const Tensor& t, const std::string& file, std::string* sidecar) {
  return Json{{"file", file}, {"offset", append_tensor(t, sidecar)},
              {"dtype", t.dtype().name()}, {"shape", t.shape()}};
}

// sidecar bytes per file name, loaded once per call
struct SidecarCache {
  fs::path dir;
  std::map<std::string, std::string> files;
  const std::string& get(const std::string& name) {
    auto it = files.find(name);
    if (it == files.end()) it = files.emplace(name, read_file(dir / name)).first;
    return it->second;
  }
};

Tensor ref_tensor(const Json& ref, SidecarCache& sc) {
  try {
    return decode_tensor(sc.get(ref.at("file").get<std::string>()), ref.at("offset").get<int64_t>(),
                         parse_dtype(ref.at("dtype").get<std::string>()),
                         ref.at("shape").get<std::vector<int64_t>>(), ref.dump());
  } catch (const IoError&) {
    throw;
  } catch (const std::exception& e) {
    throw IoError(std::string("bad tensor ref: ") + e.what());
  }
}

std::string sidecar_name(const fs::path& json_path) {
  return json_path.stem().string() + ".bin";
}

}  // namespace

uint64_t fnv1a64(const void* data, size_t size, uint64_t seed) {
  uint64_t h = seed;
  const auto* p = static_cast<const uint8_t*>(data);
  for (size_t i = 0; i < size; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

Json graph_to_json(const Graph& g, const std::string& sidecar, std::string* sidecar_bytes) {
  std::string local;
  std::string* out = sidecar_bytes ? sidecar_bytes : &local;
  out->clear();
  Json nodes = Json::array();
  for (const Node& n : g.nodes()) {
    Json jn = {{"id", n.id}, {"op", op_name(n.op)}, {"attrs", n.attrs}};
    if (!jn["attrs"].is_object()) jn["attrs"] = Json::object();
    // SPEC.md graph module: the sidecar ref {file, offset, dtype, shape}
    // lives in the constant's attrs
    if (n.payload.has_value()) jn["attrs"]["payload"] = tensor_ref(*n.payload, sidecar, out);
    nodes.push_back(std::move(jn));
  }
  Json edges = Json::array();
  for (const Edge& e : g.edges()) {
    edges.push_back({{"src", {e.src.node, e.src.port}}, {"dst", {e.dst.node, e.dst.port}}});
  }
  Json outputs = Json::array();
  for (const PortRef& o : g.outputs()) outputs.push_back({o.node, o.port});
  return Json{{"nodes", nodes}, {"edges", edges}, {"inputs", g.inputs()}, {"outputs", outputs}};
}

Graph graph_from_json(const Json& doc, const fs::path& dir) {
  SidecarCache sc{dir, {}};
  try {
    std::vector<Node> nodes;
    for (const Json& jn : doc.at("nodes")) {
      Node n;
      n.id = jn.at("id").get<NodeId>();
      n.op = parse_op(jn.at("op").get<std::string>());
      if (jn.contains("attrs") && jn.at("attrs").is_object()) n.attrs = jn.at("attrs");
      // the payload ref: attrs.payload (SPEC form), the ref keys directly in
      // attrs, or a node-level "payload" (files written by round-1 builds)
      if (n.attrs.is_object() && n.attrs.contains("payload")) {
        n.payload = ref_tensor(n.attrs.at("payload"), sc);
        n.attrs.erase("payload");
      } else if (n.attrs.is_object() && n.attrs.contains("file") && n.attrs.contains("offset") &&
                 n.attrs.contains("dtype") && n.attrs.contains("shape")) {
        n.payload = ref_tensor(n.attrs, sc);
        for (const char* k : {"file", "offset", "dtype", "shape"}) n.attrs.erase(k);
      } else if (jn.contains("payload")) {
        n.payload = ref_tensor(jn.at("payload"), sc);
      }
      nodes.push_back(std::move(n));
    }
    std::vector<Edge> edges;
    for (const Json& je : doc.at("edges")) {
      edges.push_back(Edge{PortRef{je.at("src")[0].get<NodeId>(), je.at("src")[1].get<int>()},
                           PortRef{je.at("dst")[0].get<NodeId>(), je.at("dst")[1].get<int>()}});
    }
    std::vector<PortRef> outputs;
    for (const Json& jo : doc.at("outputs")) {
      outputs.push_back(PortRef{jo[0].get<NodeId>(), jo[1].get<int>()});
    }
    return Graph(std::move(nodes), std::move(edges), doc.at("inputs").get<std::vector<NodeId>>(),
                 std::move(outputs));
  } catch (const IoError&) {
    throw;
  } catch (const std::exception& e) {
    throw IoError(std::string("malformed graph document: ") + e.what());
  }
}

void save_graph(const Graph& g, const fs::path& json_path) {
  std::string bytes;
  const std::string side = sidecar_name(json_path);
  const Json doc = graph_to_json(g, side, &bytes);
  write_file(json_path.parent_path() / side, bytes);
  write_file(json_path, doc.dump(1));
}

Graph load_graph(const fs::path& json_path) {
  return graph_from_json(parse_json(json_path), json_path.parent_path());
}

Tensor load_tensor_ref(const Json& ref, const fs::path& dir) {
  SidecarCache sc{dir, {}};
  return ref_tensor(ref, sc);
}

void save_dataset(const Dataset& dataset, const fs::path& manifest_path) {
  std::string bytes;
  const std::string side = sidecar_name(manifest_path);
  Json arr = Json::array();
  for (const Sample& s : dataset) {
    Json ins = Json::array();
    for (const Tensor& t : s.inputs) ins.push_back(tensor_ref(t, side, &bytes));
    Json js = {{"inputs", ins}};
    if (s.label.has_value()) js["label"] = *s.label;
    arr.push_back(std::move(js));
  }
  write_file(manifest_path.parent_path() / side, bytes);
  write_file(manifest_path, arr.dump(1));
}

Dataset load_dataset(const fs::path& manifest_path) {
  const Json arr = parse_json(manifest_path);
  if (!arr.is_array()) throw IoError("dataset manifest must be a JSON array");
  SidecarCache sc{manifest_path.parent_path(), {}};
  Dataset ds;
  try {
    for (const Json& js : arr) {
      Sample s;
      for (const Json& ref : js.at("inputs")) s.inputs.push_back(ref_tensor(ref, sc));
      if (js.contains("label") && !js.at("label").is_null()) s.label = js.at("label").get<int64_t>();
      ds.push_back(std::move(s));
    }
  } catch (const IoError&) {
    throw;
  } catch (const std::exception& e) {
    throw IoError(manifest_path.string() + ": malformed dataset manifest: " + e.what());
  }
  return ds;
}

void save_stats(const CalibrationStats& stats, const fs::path& path) {
  Json per = Json::object();
  for (const auto& [edge, e] : stats.per_edge) {
    per[std::to_string(edge)] = {{"min", e.min}, {"max", e.max}, {"absmax", e.absmax},
                                 {"bins", e.counts.size()}, {"counts", e.counts},
                                 {"samples", e.sample_count}};
  }
  // fingerprints as decimal strings: JSON numbers are doubles for many readers
  const Json doc = {{"dataset_fingerprint", std::to_string(stats.dataset_fingerprint)},
                    {"graph_fingerprint", std::to_string(stats.graph_fingerprint)},
                    {"per_edge", per}};
  write_file(path, doc.dump(1));
}

CalibrationStats load_stats(const fs::path& path) {
  const Json doc = parse_json(path);
  CalibrationStats st;
  if (!doc.is_object()) throw IoError(path.string() + ": stats file must be a JSON object");
  try {
    st.dataset_fingerprint = std::stoull(doc.value("dataset_fingerprint", std::string("0")));
    st.graph_fingerprint = std::stoull(doc.value("graph_fingerprint", std::string("0")));
    for (const auto& [key, j] : doc.at("per_edge").items()) {
      EdgeStats e;
      e.min = j.at("min").get<double>();
      e.max = j.at("max").get<double>();
      e.absmax = j.at("absmax").get<double>();
      e.counts = j.at("counts").get<std::vector<int64_t>>();
      e.sample_count = j.at("samples").get<int64_t>();
      if (j.contains("bins") && j.at("bins").get<size_t>() != e.counts.size()) {
        throw IoError("stats edge " + key + ": bins != len(counts)");
      }
      st.per_edge[std::stoi(key)] = std::move(e);
    }
  } catch (const IoError&) {
    throw;
  } catch (const std::exception& e) {
    throw IoError(path.string() + ": malformed stats file: " + e.what());
  }
  return st;
}

void save_strategy(const Strategy& strategy, const Json& meta, const fs::path& path) {
  Json edges = Json::object();
  for (const auto& [edge, d] : strategy.edges) {
    edges[std::to_string(edge)] = {{"bit", d.bit}, {"threshold", d.threshold}, {"sign", d.sign},
                                   {"storage_dtype", d.storage_dtype.name()},
                                   {"zero_point", d.zero_point}};
  }
  write_file(path, Json{{"meta", meta}, {"edges", edges}}.dump(1));
}

Strategy load_strategy(const fs::path& path) {
  const Json doc = parse_json(path);
  Strategy s;
  if (!doc.is_object() || !doc.contains("edges") || !doc.at("edges").is_object()) {
    throw IoError(path.string() + ": a strategy file is an object with an \"edges\" object");
  }
  try {
    const Json& edges = doc.at("edges");
    for (const auto& [key, j] : edges.items()) {
      EdgeDecision d;
      d.bit = j.at("bit").get<int>();
      d.threshold = j.at("threshold").get<double>();
      d.sign = j.at("sign").get<int>();
      d.storage_dtype = parse_dtype(j.at("storage_dtype").get<std::string>());
      d.zero_point = j.at("zero_point").get<int64_t>();
      s.edges[std::stoi(key)] = d;
    }
  } catch (const IoError&) {
    throw;
  } catch (const std::exception& e) {
    throw IoError(path.string() + ": malformed strategy file: " + e.what());
  }
  return s;
}

void save_trace(const SearchTrace& trace, const fs::path& path) {
  std::string out = trace.header.dump() + "\n";
  for (const TraceRecord& r : trace.records) {
    out += Json{{"iteration", r.iteration}, {"bits", r.bits}, {"loss", r.loss},
                {"accepted", r.accepted}}.dump();
    out += "\n";
  }
  write_file(path, out);
}

uint64_t fingerprint_graph(const Graph& g) {
  std::string bytes;
  const std::string doc = graph_to_json(g, "sidecar", &bytes).dump();
  return fnv1a64(bytes.data(), bytes.size(), fnv1a64(doc.data(), doc.size()));
}

uint64_t fingerprint_dataset(const Dataset& dataset) {
  uint64_t h = 1469598103934665603ull;
  for (const Sample& s : dataset) {
    for (const Tensor& t : s.inputs) {
      const std::string head = t.dtype().name() + shape_to_string(t.shape());
      h = fnv1a64(head.data(), head.size(), h);
      if (t.dtype().is_float()) {
        h = fnv1a64(t.floats().data(), t.floats().size() * 4, h);
      } else {
        h = fnv1a64(t.ints().data(), t.ints().size() * 4, h);
      }
    }
    const int64_t label = s.label.value_or(-1);
    h = fnv1a64(&label, sizeof(label), h);
  }
  return h;
}

}  // namespace quantc
