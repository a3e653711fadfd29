// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Minimal stand-in for boost::multiprecision::cpp_int so the reference
// sources compile here (Boost is absent from the image; SURVEY.md §8c and
// Appendix A).  The reference uses cpp_int only in space_size
// (search.cpp:69-73) and the exhaustive-search cap check (search.cpp:181):
// construction from an integer, operator*= by a small integer, comparison
// with int64, and .str() (used by our C-ABI harness).  Exact: base-1e9 limbs.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace boost {
namespace multiprecision {

class cpp_int {
 public:
  cpp_int(long long v = 0) {  // non-negative use only (products of range sizes)
    uint64_t u = v < 0 ? 0 : static_cast<uint64_t>(v);
    if (u == 0) limbs_.push_back(0);
    while (u) {
      limbs_.push_back(static_cast<uint32_t>(u % kBase));
      u /= kBase;
    }
  }
  cpp_int& operator*=(long long m) {
    uint64_t carry = 0;
    for (uint32_t& l : limbs_) {
      uint64_t cur = static_cast<uint64_t>(l) * static_cast<uint64_t>(m) + carry;
      l = static_cast<uint32_t>(cur % kBase);
      carry = cur / kBase;
    }
    while (carry) {
      limbs_.push_back(static_cast<uint32_t>(carry % kBase));
      carry /= kBase;
    }
    trim();
    return *this;
  }
  std::string str() const {
    std::string s = std::to_string(limbs_.back());
    for (size_t i = limbs_.size() - 1; i-- > 0;) {
      std::string part = std::to_string(limbs_[i]);
      s += std::string(9 - part.size(), '0') + part;
    }
    return s;
  }
  friend bool operator>(const cpp_int& a, long long b) { return a.compare(cpp_int(b)) > 0; }
  friend bool operator<(const cpp_int& a, long long b) { return a.compare(cpp_int(b)) < 0; }

 private:
  static constexpr uint64_t kBase = 1000000000ull;
  std::vector<uint32_t> limbs_;
  void trim() {
    while (limbs_.size() > 1 && limbs_.back() == 0) limbs_.pop_back();
  }
  int compare(const cpp_int& o) const {
    if (limbs_.size() != o.limbs_.size()) return limbs_.size() < o.limbs_.size() ? -1 : 1;
    for (size_t i = limbs_.size(); i-- > 0;) {
      if (limbs_[i] != o.limbs_[i]) return limbs_[i] < o.limbs_[i] ? -1 : 1;
    }
    return 0;
  }
};

}  // namespace multiprecision
}  // namespace boost
