// Philox4x32-10, host and device, with random access into a stream.
//
// The reference generator (rng.hpp:17-104) is a sequential counter PRNG:
// key = (seed lo, seed hi), counter = (0, 0, stream lo, stream hi), one
// 128-bit block per counter value, consumed as four u32 in order; next_u64 =
// lo | hi << 32 from two consecutive u32; next_double = (u64 >> 11) * 2^-53.
// Because nothing in RMAT edge draws, feature init or weight init rejects a
// draw, draw number t of a stream is a closed-form function of t:
//   block B = t / 2 with counter (B lo, B hi, stream lo, stream hi),
//   u32 pair at slots 2*(t % 2), 2*(t % 2)+1.
// That is what lets every device thread generate its own draws.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define PK_HD __host__ __device__ __forceinline__
#else
#define PK_HD inline
#endif

namespace pk {

struct Philox4 {
  uint32_t v[4];
};

PK_HD Philox4 philox_block(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                           uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
    const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
    const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return {{c0, c1, c2, c3}};
}

// Block number `b` of stream `stream` under key `seed`.
PK_HD Philox4 philox_at(uint64_t seed, uint64_t stream, uint64_t b) {
  return philox_block(static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32),
                      static_cast<uint32_t>(stream), static_cast<uint32_t>(stream >> 32),
                      static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
}

// u64 draw number t of the stream.
PK_HD uint64_t philox_u64_at(uint64_t seed, uint64_t stream, uint64_t t) {
  const Philox4 blk = philox_at(seed, stream, t >> 1);
  const int s = static_cast<int>(t & 1) * 2;
  return static_cast<uint64_t>(blk.v[s]) | (static_cast<uint64_t>(blk.v[s + 1]) << 32);
}

PK_HD double u64_to_unit(uint64_t x) { return static_cast<double>(x >> 11) * 0x1.0p-53; }

// Sequential host generator with the reference's consumption order, used
// for the permutation pair (Fisher-Yates with rejection; graph.hpp:84-93).
struct PhiloxStream {
  uint64_t seed, stream, block = 0;
  Philox4 cur{};
  int pos = 4;
  PhiloxStream(uint64_t s, uint64_t st) : seed(s), stream(st) {}
  uint32_t next_u32() {
    if (pos == 4) {
      cur = philox_at(seed, stream, block++);
      pos = 0;
    }
    return cur.v[pos++];
  }
  uint64_t next_u64() {
    const uint64_t lo = next_u32();
    const uint64_t hi = next_u32();
    return (hi << 32) | lo;
  }
  uint64_t randint(uint64_t bound) {
    const uint64_t threshold = (~bound + 1) % bound;
    for (;;) {
      const uint64_t r = next_u64();
      if (r >= threshold) return r % bound;
    }
  }
};

}  // namespace pk
