// hostdev.h — code shared verbatim by the device scheduler and the host build
// used in CPU tests (no CUDA headers required when compiled by g++).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define PPSD_HD __host__ __device__ __forceinline__
#else
#define PPSD_HD inline
#endif

namespace ppsd {

// splitmix64 finalizer — reference rng.py:29-37
PPSD_HD uint64_t hmix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
constexpr uint64_t kGoldenGamma = 0x9E3779B97F4A7C15ull;

// RngStream(seed, counter=c).uniform() — rng.py:81-85 (exact: integer hash,
// then an exact int->double conversion and a power-of-two scale)
PPSD_HD double counter_uniform(uint64_t seed, uint64_t c) {
  return (double)(hmix64(seed + (c + 1) * kGoldenGamma) >> 11) * 0x1p-53;
}

// derive_seed(seed, label) for a string label — rng.py:51-63
PPSD_HD uint64_t derive_seed_str(uint64_t seed, const char* label) {
  uint64_t h = hmix64(seed ^ 0xA24BAED4963EE407ull);
  for (const char* c = label; *c; ++c) h = hmix64(h ^ ((uint64_t)(unsigned char)*c + 1));
  return h;
}

// ToyLM salts — toylm.py:25-29
constexpr uint64_t kSeqSalt = 0x243F6A8885A308D3ull;
constexpr uint64_t kTokenSalt = 0x13198A2E03707344ull;
constexpr uint64_t kLayerSalt = 0x452821E638D01377ull;
constexpr uint64_t kLogitSalt = 0xBE5466CF34E90C6Cull;
constexpr uint64_t kNoiseSalt = 0xC0AC29B7C97C50DDull;

// ToyLM.extend_digest (toylm.py:76-80)
PPSD_HD uint64_t toy_extend(uint64_t d, int tok) {
  return hmix64(d ^ (kTokenSalt + (uint64_t)(int64_t)tok));
}
// ToyLM.advance_digest (toylm.py:88-96): layers a+1..b
PPSD_HD uint64_t toy_advance(uint64_t d, int a, int b) {
  for (int k = a + 1; k <= b; ++k) d = hmix64(d ^ ((uint64_t)k * kLayerSalt));
  return d;
}

}  // namespace ppsd
