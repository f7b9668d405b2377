// fuseplan-b200 — counter-based RNG shared by kernels and host code.
//
// Philox4x32-10 (Salmon et al., SC'11) for per-sample sampling streams and a
// splitmix64-style hash for deterministic synthetic weights / prompts. Both
// are plain integer arithmetic so the numpy oracle (oracle/model_oracle.py)
// reproduces every bit.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define FP_HD __host__ __device__ __forceinline__
#else
#define FP_HD inline
#endif

namespace fpk {

struct U4 {
  uint32_t x, y, z, w;
};

FP_HD void mulhilo32(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
  const uint64_t p = static_cast<uint64_t>(a) * b;
  hi = static_cast<uint32_t>(p >> 32);
  lo = static_cast<uint32_t>(p);
}

// counter c, key k -> 4 random words
FP_HD U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#ifdef __CUDACC__
#pragma unroll
#endif
  for (int i = 0; i < 10; ++i) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(0xD2511F53u, c.x, hi0, lo0);
    mulhilo32(0xCD9E8D57u, c.z, hi1, lo1);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// splitmix64 finaliser of a (seed, tag, index) triple.
FP_HD uint64_t hash3(uint64_t seed, uint64_t tag, uint64_t index) {
  uint64_t z = seed ^ (tag * 0xD1B54A32D192ED03ull);
  z += (index + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// 24-bit uniform in [0, 1).
FP_HD float unit24(uint64_t h) { return static_cast<float>(h >> 40) * (1.0f / 16777216.0f); }

// Tags of the synthetic tensors: (model << 24) | (layer << 8) | kind.
enum : uint32_t {
  kTagEmbed = 1, kTagWqkv = 2, kTagWo = 3, kTagWgu = 4, kTagWd = 5, kTagAttnNorm = 6, kTagMlpNorm = 7,
  kTagFinalNorm = 8, kTagHead = 9, kTagValueHead = 10, kTagPrompt = 0xF1, kTagResponse = 0xF2
};

FP_HD uint64_t weight_tag(uint32_t model, uint32_t layer, uint32_t kind) {
  return (static_cast<uint64_t>(model) << 24) | (static_cast<uint64_t>(layer) << 8) | kind;
}

}  // namespace fpk
