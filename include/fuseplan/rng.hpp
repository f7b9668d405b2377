// fuseplan-b200 — deterministic host RNG used for sample lengths.
//
// Bit-identical to the reference generator (proj/include/fuseplan/rng.hpp:10-54,
// Box-Muller at proj/src/core.cpp:95-108): lengths drawn here must equal the
// reference's for the same seed, because sample-to-GPU assignment and every
// migration decision depend on them. <random> is avoided for the same reason
// the reference gives: its distributions are implementation-defined.
#pragma once

#include <cstdint>

namespace fuseplan {

/// One splitmix64 step: advances `state` by the golden-ratio increment and
/// returns the finalised mix of the new state.
inline std::uint64_t splitmix64(std::uint64_t& state) {
  constexpr std::uint64_t kGamma = 0x9e3779b97f4a7c15ull;
  constexpr std::uint64_t kMul1 = 0xbf58476d1ce4e5b9ull;
  constexpr std::uint64_t kMul2 = 0x94d049bb133111ebull;
  state += kGamma;
  std::uint64_t x = state;
  x = (x ^ (x >> 30)) * kMul1;
  x = (x ^ (x >> 27)) * kMul2;
  return x ^ (x >> 31);
}

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : s_(seed) {}

  std::uint64_t next_u64() { return splitmix64(s_); }

  /// Uniform integer in [0, n) by 128-bit multiply-high (n > 0).
  std::uint64_t next_below(std::uint64_t n) {
    const unsigned __int128 wide = static_cast<unsigned __int128>(next_u64()) * n;
    return static_cast<std::uint64_t>(wide >> 64);
  }

  /// Uniform double in [0, 1) from the top 53 bits.
  double next_double() {
    constexpr double kInv53 = 1.0 / 9007199254740992.0;  // 2^-53
    return static_cast<double>(next_u64() >> 11) * kInv53;
  }

  /// Standard normal (polar-free Box-Muller); draws come in pairs, the sine
  /// branch is served on the next call.
  double next_normal();

 private:
  std::uint64_t s_;
  double spare_ = 0.0;
  bool have_spare_ = false;
};

/// Independent stream `stream` of a master seed (reference rng.hpp:49-54).
inline std::uint64_t derive_seed(std::uint64_t master, std::uint64_t stream) {
  std::uint64_t st = master ^ (0xd1b54a32d192ed03ull * (stream + 1));
  const std::uint64_t hi = splitmix64(st);
  const std::uint64_t lo = splitmix64(st);
  return hi ^ (lo << 1) ^ (lo >> 63);
}

}  // namespace fuseplan
