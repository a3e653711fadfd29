// quantc/fixtures.hpp — deterministic synthetic models, datasets and hardware
// specs (B200 build).
//
// Drop-in for /root/reference/proj/include/quantc/fixtures.hpp:13-60, which
// the reference declares without an implementation; the contract is
// SPEC.md:734-782 (fixtures module).  Generation is deterministic from the
// seed: std::mt19937_64 with an explicit Box-Muller normal (no
// implementation-defined std:: distributions), so the bytes are identical on
// every platform.  The generators compute what they verify (centroid head,
// overflow margins) with a small host forward in the reference's arithmetic
// (double accumulation, one rounding to float); that is generation-time
// bookkeeping, not the hot path.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "quantc/graph.hpp"
#include "quantc/hwspec.hpp"
#include "quantc/interpreter.hpp"

namespace quantc {
namespace fixtures {

// reference fixtures.hpp:16-20
struct ModelFixture {
  Graph graph;
  Dataset calibration;
  Dataset evaluation;
};

// reference fixtures.hpp:22-26.  Three 3x3 conv2d (+relu) over 8x8x3 inputs,
// global average pooling, flatten, a 10-class dense head set to the class
// centroids of the pooled features of a held-out 256-sample training draw
// (nearest-centroid scores, centred on the mean centroid); 64 calibration and
// 256 evaluation samples from a seeded 10-prototype mixture, each drawn with a
// verified margin: its fp32 top-1 beats the runner-up by > 5% of the score
// scale (rejection sampling), so realized low-bit models keep the top-1.
ModelFixture make_small_cnn(uint64_t seed = 7);

// reference fixtures.hpp:28-33.  One dense layer with a 512-wide reduction
// (inputs in [0, 1), zero-mean weights).  Verified at generation time with
// max-calibrated thresholds: 8 effective bits overflow int16 accumulation on
// the calibration data, 6 effective bits stay below 2^15 with margin.
ModelFixture make_overflow_probe(uint64_t seed = 11);

// reference fixtures.hpp:35-40: fig3, x86_vnni_like, arm_vmlal_like,
// int8_int32.  Unknown names throw FixtureError.
HardwareSpec spec_fixture(const std::string& name);

// reference fixtures.hpp:42-44.  dense/relu chain with exactly
// `searchable_edges` quantizable edges under int8_int32 (a dense contributes
// its data and weight edges, a relu its data edge).
Graph make_deep_chain(int searchable_edges, uint64_t seed = 3);

// reference fixtures.hpp:46-48.  conv2d -> add(constant) -> global_avg_pool2d
// (the Fig. 4 chain), 16 calibration + 16 evaluation samples.
ModelFixture make_conv_add_pool_chain(uint64_t seed = 5);

// reference fixtures.hpp:50-53
class FixtureError : public std::runtime_error {
 public:
  explicit FixtureError(const std::string& what) : std::runtime_error(what) {}
};

// reference fixtures.hpp:55-56.  Graph files (+ sidecars), dataset
// manifests and spec files of every committed fixture under dir.
void write_all(const std::string& dir);

// reference fixtures.hpp:58-60.  Regenerates into a scratch directory and
// byte-compares every file (and the file set) against dir.
void verify_committed(const std::string& dir);

}  // namespace fixtures
}  // namespace quantc
