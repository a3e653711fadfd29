// quantc/topology.hpp — Algorithm 1 and simulated_quantize insertion
// (B200 build; host-side graph passes run once per model).
//
// Drop-in for /root/reference/proj/include/quantc/topology.hpp.
#pragma once

#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "quantc/graph.hpp"
#include "quantc/hwspec.hpp"

namespace quantc {

// reference topology.hpp:16-27
struct Topology {
  std::set<NodeId> qv;
  std::set<NodeId> nqv;
  std::map<int, std::vector<DType>> edge_dtypes;
  std::map<int, DType> fixed_edges;

  bool is_quantized(NodeId id) const { return qv.count(id) > 0; }
};

class TopologyError : public std::runtime_error {
 public:
  explicit TopologyError(const std::string& what) : std::runtime_error(what) {}
};

Topology generate_topology(const Graph& g, const HardwareSpec& spec);
Graph insert_simulated_quantize(const Graph& g, const Topology& t);

// reference topology.hpp:50-62
struct Segment {
  std::vector<NodeId> vertices;
  std::vector<Edge> interior_edges;
  std::vector<Edge> boundary_edges;
};

struct Partition {
  std::vector<Segment> segments;
  std::vector<NodeId> remainder;
  std::vector<Edge> remainder_edges;
};

Partition partition_segments(const Graph& g, const Topology& t);
std::vector<int> searchable_edge_indices(const Topology& t);
std::vector<int> simulated_edge_indices(const Graph& g, const Topology& t);
std::string dump_topology(const Graph& g, const Topology& t);

}  // namespace quantc
