// genome.hpp -- the offload pattern: one bit per candidate loop, 1 = run that loop on the GPU.
//
// API-compatible with acctune::Genome (/root/reference/proj/include/acctune/genome.hpp:18-73):
// a value type over std::vector<uint8_t> of 0/1 (gene 0 first), string form "101000011000",
// lexicographic order (== bit-string order), FNV-1a hash over the bit bytes.  bits().data() is
// what crosses the C ABI (include/mmx.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

#include "mmxhost/errors.hpp"

namespace mmxhost {

class Genome {
 public:
  using Bits = std::vector<std::uint8_t>;

  Genome() = default;
  explicit Genome(Bits bits) : bits_(std::move(bits)) {}

  static Genome zeros(std::size_t n) { return Genome(Bits(n, std::uint8_t{0})); }
  static Genome ones(std::size_t n) { return Genome(Bits(n, std::uint8_t{1})); }

  // Accepts only '0' and '1' (genome.hpp:26-34).
  static Genome from_string(std::string_view text) {
    Bits bits(text.size());
    for (std::size_t k = 0; k < text.size(); ++k) {
      if (text[k] == '1') bits[k] = 1;
      else if (text[k] == '0') bits[k] = 0;
      else throw Error("genome string must be over {0,1}: " + std::string(text));
    }
    return Genome(std::move(bits));
  }

  std::string to_string() const {
    std::string out;
    out.reserve(bits_.size());
    for (std::uint8_t b : bits_) out.push_back(b ? '1' : '0');
    return out;
  }

  std::size_t size() const { return bits_.size(); }
  bool empty() const { return bits_.empty(); }
  bool test(std::size_t k) const { return bits_[k] != 0; }
  void set(std::size_t k, bool v) { bits_[k] = v ? 1 : 0; }
  void flip(std::size_t k) { bits_[k] = bits_[k] ? 0 : 1; }
  std::size_t count() const {
    std::size_t ones = 0;
    for (std::uint8_t b : bits_) ones += b != 0;
    return ones;
  }
  const Bits& bits() const { return bits_; }

  // lexicographic, shorter-is-smaller on a common prefix: the order std::vector gives
  friend bool operator==(const Genome& x, const Genome& y) { return x.bits_ == y.bits_; }
  friend bool operator!=(const Genome& x, const Genome& y) { return !(x == y); }
  friend bool operator<(const Genome& x, const Genome& y) { return x.bits_ < y.bits_; }
  friend bool operator>(const Genome& x, const Genome& y) { return y < x; }
  friend bool operator<=(const Genome& x, const Genome& y) { return !(y < x); }
  friend bool operator>=(const Genome& x, const Genome& y) { return !(x < y); }

  // FNV-1a, 64-bit, over the bit bytes (genome.hpp:59-69)
  struct Hash {
    std::size_t operator()(const Genome& g) const {
      std::uint64_t h = 0xcbf29ce484222325ull;
      for (std::uint8_t b : g.bits_) h = (h ^ b) * 0x100000001b3ull;
      return static_cast<std::size_t>(h);
    }
  };

 private:
  Bits bits_;
};

}  // namespace mmxhost
