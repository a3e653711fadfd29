// quantc/bigint.hpp — exact unsigned integer for search-space sizes.
//
// Stands in for boost::multiprecision::cpp_int in the one place the reference
// API uses it (search.hpp:72 space_size; paper §5.3 "larger than 4^118").
// Supports what callers of space_size use: construction from an integer,
// *= small factor, comparison with integers and other BigUInt, str().
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace quantc {

class BigUInt {
 public:
  BigUInt(uint64_t v = 0);
  BigUInt& operator*=(uint64_t m);
  std::string str() const;
  int compare(const BigUInt& o) const;

  friend bool operator==(const BigUInt& a, const BigUInt& b) { return a.compare(b) == 0; }
  friend bool operator<(const BigUInt& a, const BigUInt& b) { return a.compare(b) < 0; }
  friend bool operator>(const BigUInt& a, const BigUInt& b) { return a.compare(b) > 0; }
  friend bool operator>(const BigUInt& a, long long b) { return a.compare(from_signed(b)) > 0; }
  friend bool operator<(const BigUInt& a, long long b) { return a.compare(from_signed(b)) < 0; }
  friend bool operator==(const BigUInt& a, long long b) { return a.compare(from_signed(b)) == 0; }

 private:
  static BigUInt from_signed(long long v) { return BigUInt(v < 0 ? 0 : static_cast<uint64_t>(v)); }
  std::vector<uint32_t> limbs_;  // base 2^32, little-endian, no leading zeros except "0"
};

}  // namespace quantc
