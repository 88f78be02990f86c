// Keyed random streams, bit-exact with the reference's RNG contract.
//
// The reference draws every partitioning decision from
//   np.random.default_rng(np.random.SeedSequence(seed, spawn_key=key))
// (pkg/src/syscd/partitioning.py:30-38) and consumes it through
// Generator.permutation (partitioning.py:95,107,117) and Generator.integers
// (solvers.py:159-166,326-333).  numpy is an unvendored third-party dependency
// (numpy 2.3.5 in this image, pyproject.toml:10-13 pins only >=1.24); this file
// restates its published algorithms:
//   * SeedSequence entropy assembly + hashmix pool (numpy/random/bit_generator.pyx)
//   * PCG64 = pcg_setseq_128_xsl_rr_64 with numpy's 32-bit output buffering
//   * Generator.permutation = Fisher-Yates from the top with masked rejection
//     (random_interval, numpy/random/src/distributions/distributions.c)
//   * Generator.integers(lo, hi) for int64 = Lemire bounded draw on 32-bit
//     words when the range fits (random_bounded_uint64_fill, use_masked=False)
// Everything is __host__ __device__ so the same code backs the host KAT entry
// point (syscd_rng_permutation) and the device planning kernels (plan.cu).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define SYSCD_HD __host__ __device__ __forceinline__
#else
#define SYSCD_HD static inline
#endif

namespace syscd {

struct U128 {
  uint64_t hi, lo;
};

SYSCD_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

SYSCD_HD U128 u128_mul(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = mulhi64(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
  return r;
}

SYSCD_HD U128 u128_add(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1u : 0u);
  return r;
}

// SeedSequence hash constants.
constexpr uint32_t kInitA = 0x43b0d7e5u;
constexpr uint32_t kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu;
constexpr uint32_t kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu;
constexpr uint32_t kMixR = 0x4973f715u;
constexpr int kPool = 4;
constexpr int kMaxEntropyWords = 16;

SYSCD_HD uint32_t ss_hashmix(uint32_t value, uint32_t* hc) {
  value ^= *hc;
  *hc *= kMultA;
  value *= *hc;
  value ^= value >> 16;
  return value;
}

SYSCD_HD uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> 16;
  return r;
}

// Append the little-endian 32-bit limbs of v (0 -> a single zero limb).
SYSCD_HD int ss_push_words(uint32_t* w, int n, uint64_t v) {
  if (v == 0) {
    w[n++] = 0;
    return n;
  }
  while (v != 0 && n < kMaxEntropyWords) {
    w[n++] = (uint32_t)(v & 0xffffffffu);
    v >>= 32;
  }
  return n;
}

// PCG64 with numpy's buffered 32-bit draws.
struct Pcg64 {
  U128 state;
  U128 inc;
  uint32_t buf32;
  int has32;
};

SYSCD_HD void pcg_step(Pcg64* g) {
  const U128 mult = {0x2360ed051fc65da4ull, 0x4385df649fccf645ull};
  g->state = u128_add(u128_mul(g->state, mult), g->inc);
}

SYSCD_HD uint64_t pcg_next64(Pcg64* g) {
  pcg_step(g);
  uint64_t x = g->state.hi ^ g->state.lo;
  unsigned rot = (unsigned)(g->state.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

SYSCD_HD uint32_t pcg_next32(Pcg64* g) {
  if (g->has32) {
    g->has32 = 0;
    return g->buf32;
  }
  uint64_t v = pcg_next64(g);
  g->has32 = 1;
  g->buf32 = (uint32_t)(v >> 32);
  return (uint32_t)(v & 0xffffffffu);
}

// default_rng(SeedSequence(seed, spawn_key=key)).
SYSCD_HD void pcg_seed_keyed(Pcg64* g, uint64_t seed, const uint64_t* key, int key_len) {
  uint32_t ent[kMaxEntropyWords];
  int n = ss_push_words(ent, 0, seed);
  if (key_len > 0) {
    while (n < kPool) ent[n++] = 0;  // pad run entropy to the pool size
    for (int i = 0; i < key_len; ++i) n = ss_push_words(ent, n, key[i]);
  }
  uint32_t pool[kPool];
  uint32_t hc = kInitA;
  for (int i = 0; i < kPool; ++i) pool[i] = ss_hashmix(i < n ? ent[i] : 0u, &hc);
  for (int s = 0; s < kPool; ++s)
    for (int d = 0; d < kPool; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
  for (int s = kPool; s < n; ++s)
    for (int d = 0; d < kPool; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], &hc));
  // generate_state(4, uint64): 8 words cycling over the pool.
  uint32_t st[8];
  uint32_t hb = kInitB;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    st[i] = v;
  }
  uint64_t s0 = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  uint64_t s1 = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
  uint64_t s2 = (uint64_t)st[4] | ((uint64_t)st[5] << 32);
  uint64_t s3 = (uint64_t)st[6] | ((uint64_t)st[7] << 32);
  U128 initstate = {s0, s1};
  U128 initseq = {s2, s3};
  g->inc.hi = (initseq.hi << 1) | (initseq.lo >> 63);
  g->inc.lo = (initseq.lo << 1) | 1u;
  g->state.hi = 0;
  g->state.lo = 0;
  pcg_step(g);
  g->state = u128_add(g->state, initstate);
  pcg_step(g);
  g->has32 = 0;
  g->buf32 = 0;
}

SYSCD_HD void pcg_seed3(Pcg64* g, uint64_t seed, uint64_t k0, uint64_t k1, uint64_t k2, int key_len) {
  uint64_t key[3] = {k0, k1, k2};
  pcg_seed_keyed(g, seed, key, key_len);
}

// random_interval(max): uniform in [0, max] by masked rejection.
SYSCD_HD uint64_t pcg_interval(Pcg64* g, uint64_t max) {
  if (max == 0) return 0;
  uint64_t mask = max;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  mask |= mask >> 32;
  uint64_t value;
  if (max <= 0xffffffffull) {
    while ((value = (pcg_next32(g) & (uint32_t)mask)) > max) {
    }
  } else {
    while ((value = (pcg_next64(g) & mask)) > max) {
    }
  }
  return value;
}

// Generator.integers(lo, hi) for the default int64 dtype, hi > lo.
SYSCD_HD int64_t pcg_integers(Pcg64* g, int64_t lo, int64_t hi) {
  uint64_t rng = (uint64_t)(hi - lo - 1);
  if (rng == 0) return lo;
  if (rng <= 0xffffffffull) {
    if (rng == 0xffffffffull) return lo + (int64_t)pcg_next32(g);
    uint32_t rng_excl = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)pcg_next32(g) * rng_excl;
    uint32_t left = (uint32_t)(m & 0xffffffffu);
    if (left < rng_excl) {
      uint32_t threshold = (uint32_t)((0xffffffffu - (uint32_t)rng) % rng_excl);
      while (left < threshold) {
        m = (uint64_t)pcg_next32(g) * rng_excl;
        left = (uint32_t)(m & 0xffffffffu);
      }
    }
    return lo + (int64_t)(m >> 32);
  }
  // 64-bit Lemire (ranges beyond 2^32 never occur for coordinate counts here).
  if (rng == 0xffffffffffffffffull) return lo + (int64_t)pcg_next64(g);
  uint64_t rng_excl = rng + 1;
  uint64_t x = pcg_next64(g);
  uint64_t mlo = x * rng_excl, mhi = mulhi64(x, rng_excl);
  if (mlo < rng_excl) {
    uint64_t threshold = (0xffffffffffffffffull - rng) % rng_excl;
    while (mlo < threshold) {
      x = pcg_next64(g);
      mlo = x * rng_excl;
      mhi = mulhi64(x, rng_excl);
    }
  }
  return lo + (int64_t)mhi;
}

// Generator.permutation(n) applied in place to `a` (caller fills a[i] = i or
// any payload): for i = n-1 .. 1 swap a[i], a[random_interval(i)].
template <typename T>
SYSCD_HD void pcg_shuffle(Pcg64* g, T* a, int64_t n) {
  for (int64_t i = n - 1; i >= 1; --i) {
    int64_t j = (int64_t)pcg_interval(g, (uint64_t)i);
    T t = a[i];
    a[i] = a[j];
    a[j] = t;
  }
}

}  // namespace syscd
