// NumPy-exact Generator(Philox(seed)) for PARITY mode (plas.py:240-262).
//
// NumPy 2.3.5: SeedSequence(seed).generate_state(2, uint64) -> Philox4x64-10
// key; the 256-bit counter is incremented before each block; 64-bit words are
// consumed in order and next_uint32 serves the low half first and buffers the
// high half.  integers(0, b) is 32-bit Lemire rejection; permutation(n) is a
// Fisher-Yates shuffle i = n-1 .. 1 with masked rejection.  Pinned against
// NumPy itself in tests/test_host_logic.py.
#pragma once
#include <stdint.h>
#include <string.h>

#include "common.cuh"

namespace plas {
namespace host {

inline void seed_key(uint64_t seed, uint64_t key[2]) {
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu,
                 MULT_B = 0x58f38dedu, MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t ent[2];
  int nent = 0;
  if (seed == 0) ent[nent++] = 0;
  while (seed) {
    ent[nent++] = (uint32_t)seed;
    seed >>= 32;
  }
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    v ^= v >> 16;
    return v;
  };
  auto mix = [&](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; i++) pool[i] = hashmix(i < nent ? ent[i] : 0u);
  for (int s = 0; s < 4; s++)
    for (int d = 0; d < 4; d++)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < nent; s++)
    for (int d = 0; d < 4; d++) pool[d] = mix(pool[d], hashmix(ent[s]));
  uint32_t hb = INIT_B, st[4];
  for (int i = 0; i < 4; i++) {
    uint32_t v = pool[i] ^ hb;
    hb *= MULT_B;
    v *= hb;
    st[i] = v ^ (v >> 16);
  }
  key[0] = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  key[1] = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
}

struct NumpyPhilox {
  unsigned long long ctr[4], key[2], buf[4];
  int pos, has32;
  uint32_t u32;

  void seed(uint64_t s) {
    memset(this, 0, sizeof(*this));
    uint64_t k[2];
    seed_key(s, k);
    key[0] = k[0];
    key[1] = k[1];
    pos = 4;
  }
  uint64_t next64() {
    if (pos < 4) return buf[pos++];
    for (int i = 0; i < 4; i++)
      if (++ctr[i]) break;
    philox4x64_10(ctr, key[0], key[1], buf);
    pos = 1;
    return buf[0];
  }
  uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    uint64_t v = next64();
    has32 = 1;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  // Generator.integers(0, high), 1 <= high <= 2^32
  int64_t integers(int64_t high) {
    uint64_t rng = (uint64_t)(high - 1);
    if (rng == 0) return 0;
    if (rng == 0xffffffffull) return next32();
    uint32_t ex = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)next32() * ex;
    uint32_t left = (uint32_t)m;
    if (left < ex) {
      uint32_t th = (uint32_t)(0xffffffffu - (uint32_t)rng) % ex;
      while (left < th) {
        m = (uint64_t)next32() * ex;
        left = (uint32_t)m;
      }
    }
    return (int64_t)(m >> 32);
  }
  // Generator.permutation(n) into T out[n]
  template <typename T>
  void permutation(int64_t n, T* out) {
    for (int64_t i = 0; i < n; i++) out[i] = (T)i;
    for (int64_t i = n - 1; i >= 1; i--) {
      uint64_t mask = (uint64_t)i;
      mask |= mask >> 1;
      mask |= mask >> 2;
      mask |= mask >> 4;
      mask |= mask >> 8;
      mask |= mask >> 16;
      mask |= mask >> 32;
      uint64_t v;
      if ((uint64_t)i <= 0xffffffffull) {
        do {
          v = next32() & mask;
        } while (v > (uint64_t)i);
      } else {
        do {
          v = next64() & mask;
        } while (v > (uint64_t)i);
      }
      T t = out[i];
      out[i] = out[v];
      out[v] = t;
    }
  }
};

}  // namespace host
}  // namespace plas
