// Drop-in check of include/quantc/fixtures.hpp (reference fixtures.hpp:13-60,
// SPEC.md:734-782) from a C++ program built against the B200 library: the
// header compiles as the reference declares it, generation is deterministic,
// every fixture validates, the spec fixtures parse, the 118-edge chain has
// the paper's search-space size, and write_all / verify_committed round-trip
// (and catch a changed byte).   usage: fixtures_check <scratch dir> [<committed dir>]
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <string>

#include "quantc/fixtures.hpp"
#include "quantc/search.hpp"
#include "quantc/serialize.hpp"
#include "quantc/topology.hpp"

using namespace quantc;

#define CHECK(c)                                                         \
  do {                                                                   \
    if (!(c)) {                                                          \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                          \
    }                                                                    \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  namespace fs = std::filesystem;
  const fs::path dir(argv[1]);
  const auto a = fixtures::make_small_cnn();
  const auto b = fixtures::make_small_cnn(7);
  CHECK(fingerprint_graph(a.graph) == fingerprint_graph(b.graph));
  CHECK(fingerprint_dataset(a.calibration) == fingerprint_dataset(b.calibration));
  CHECK(fingerprint_dataset(a.evaluation) == fingerprint_dataset(b.evaluation));
  CHECK(fingerprint_graph(fixtures::make_small_cnn(8).graph) != fingerprint_graph(a.graph));
  CHECK(a.calibration.size() == 64 && a.evaluation.size() == 256);
  CHECK(validate_graph(a.graph).empty());
  const auto probe = fixtures::make_overflow_probe();
  CHECK(validate_graph(probe.graph).empty());
  CHECK(probe.calibration.size() == 64 && probe.calibration[0].inputs[0].shape()[1] == 512);
  const auto chain = fixtures::make_conv_add_pool_chain();
  CHECK(validate_graph(chain.graph).empty());
  for (const char* s : {"fig3", "x86_vnni_like", "arm_vmlal_like", "int8_int32"}) {
    CHECK(!fixtures::spec_fixture(s).table().empty());
  }
  CHECK(fixtures::spec_fixture("arm_vmlal_like").signatures(OpKind::kConv2d).size() == 2);
  bool threw = false;
  try {
    fixtures::spec_fixture("tpu");
  } catch (const fixtures::FixtureError&) {
    threw = true;
  }
  CHECK(threw);
  // SPEC.md acceptance 9: the 118-edge graph's space exceeds 4^118
  const Graph deep = fixtures::make_deep_chain(118);
  CHECK(validate_graph(deep).empty());
  const HardwareSpec i8 = fixtures::spec_fixture("int8_int32");
  const Topology topo = generate_topology(deep, i8);
  CHECK(searchable_edge_indices(topo).size() == 118);
  BigUInt four118(1);
  for (int i = 0; i < 118; ++i) four118 *= 4;
  CHECK(space_size(build_search_space(deep, topo, i8)) > four118);
  // committed files: write, verify, then a changed byte must be caught
  fixtures::write_all(dir.string());
  fixtures::verify_committed(dir.string());
  if (argc > 2) fixtures::verify_committed(argv[2]);  // the repo's committed copy
  {
    std::fstream f(dir / "small_cnn.json", std::ios::in | std::ios::out | std::ios::binary);
    f.seekp(10);
    f.put('#');
  }
  threw = false;
  try {
    fixtures::verify_committed(dir.string());
  } catch (const fixtures::FixtureError&) {
    threw = true;
  }
  CHECK(threw);
  std::printf("ok\n");
  return 0;
}
