// rng.hpp -- the GA's random source.  The draw discipline is part of the contract
// (/root/reference/proj/include/acctune/rng.hpp:13-31): std::mt19937_64, exactly one engine
// step per helper call, no std::uniform_*_distribution (library-dependent sequences).
#pragma once

#include <cstddef>
#include <cstdint>
#include <random>

namespace mmxhost {

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : engine_(seed) {}

  std::uint64_t raw() { return engine_(); }
  // low bit of one draw
  bool bit() { return (raw() & 1u) == 1u; }
  // top 53 bits of one draw scaled into [0, 1)
  double real01() { return static_cast<double>(raw() >> 11) * (1.0 / 9007199254740992.0); }
  // one draw modulo n
  std::size_t index(std::size_t n) { return static_cast<std::size_t>(raw() % n); }

 private:
  std::mt19937_64 engine_;
};

}  // namespace mmxhost
