// Round trips of the C++-only serialize.hpp files (dataset manifest, strategy,
// trace) against the B200 library; built and run by tests/test_serialize.py.
// Reference: proj/include/quantc/serialize.hpp:36-50.
#include <algorithm>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <string>

#include "quantc/serialize.hpp"

using namespace quantc;

#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                    \
    }                                                              \
  } while (0)

int main(int argc, char** argv) {
  const std::filesystem::path dir = argc > 1 ? argv[1] : ".";
  // dataset: fp32 and int8 inputs, with and without labels
  Dataset ds;
  ds.push_back(Sample{{Tensor::from_floats({2, 3}, {1.5f, -0.f, 3e-38f, 7.f, -1e30f, 0.1f})}, 4});
  ds.push_back(Sample{{Tensor::from_ints(parse_dtype("int8"), {3}, {-128, 0, 127}),
                       Tensor::from_floats({1}, {2.f})}, std::nullopt});
  save_dataset(ds, dir / "data.json");
  CHECK(std::filesystem::exists(dir / "data.bin"));
  CHECK(std::filesystem::file_size(dir / "data.bin") == 6 * 4 + 3 + 4);  // natural widths
  const Dataset back = load_dataset(dir / "data.json");
  CHECK(back.size() == 2);
  CHECK(back[0].label == std::optional<int64_t>(4) && !back[1].label.has_value());
  CHECK(std::ranges::equal(back[0].inputs[0].floats(), ds[0].inputs[0].floats()));
  CHECK(back[1].inputs[0].dtype() == parse_dtype("int8"));
  CHECK(std::ranges::equal(back[1].inputs[0].ints(), ds[1].inputs[0].ints()));
  CHECK(fingerprint_dataset(back) == fingerprint_dataset(ds));

  // strategy
  Strategy s;
  s.edges[3] = EdgeDecision{8, 0.25, 1, 0, parse_dtype("int8")};
  s.edges[11] = EdgeDecision{4, 6.0, 0, 7, parse_dtype("uint8")};
  save_strategy(s, Json{{"spec", "int8_int32"}}, dir / "strategy.json");
  const Strategy s2 = load_strategy(dir / "strategy.json");
  CHECK(s2.edges.size() == 2);
  for (const auto& [k, d] : s.edges) {
    const EdgeDecision& e = s2.edges.at(k);
    CHECK(e.bit == d.bit && e.threshold == d.threshold && e.sign == d.sign &&
          e.zero_point == d.zero_point && e.storage_dtype == d.storage_dtype);
  }

  // trace: header line first, then one record per line
  SearchTrace t;
  t.header = Json{{"graph", "g"}, {"edges", 2}};
  t.records.push_back(TraceRecord{0, {8, 8}, 0.0, true});
  t.records.push_back(TraceRecord{1, {6, 8}, 0.125, false});
  save_trace(t, dir / "trace.jsonl");
  std::ifstream f(dir / "trace.jsonl");
  std::string line;
  int n = 0;
  while (std::getline(f, line)) {
    const Json j = Json::parse(line);
    if (n == 0) CHECK(j == t.header);
    else CHECK(j.at("iteration").get<int64_t>() == n - 1 &&
               j.at("bits").get<std::vector<int>>() == t.records[n - 1].bits);
    ++n;
  }
  CHECK(n == 3);

  // malformed files are IoError
  std::ofstream(dir / "bad.json") << "[1,";
  bool threw = false;
  try {
    load_strategy(dir / "bad.json");
  } catch (const IoError&) {
    threw = true;
  }
  CHECK(threw);
  std::puts("serialize round trip ok");
  return 0;
}
