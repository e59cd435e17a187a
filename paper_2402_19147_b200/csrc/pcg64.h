// numpy-compatible random stream for the QMCUR index draw.
//
// The reference draws its indices from `np.random.default_rng(plan.seed)`
// (cur.py:251) and consumes one `Generator.random()` double per draw
// (cur.py:235).  default_rng(seed) is PCG64 (XSL-RR 128/64) seeded through
// numpy's SeedSequence; random() is (next_uint64 >> 11) * 2^-53.  This header
// restates those published algorithms (numpy 2.x, bit_generator.pyx
// SeedSequence + pcg64.h) so the uniforms can be produced on the device with
// no host round trip.  Everything here is plain integer arithmetic usable from
// host C++ and CUDA device code alike.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define QCUR_HD __host__ __device__ __forceinline__
#else
#define QCUR_HD inline
#endif

namespace qcur {

struct u128 {
  uint64_t hi, lo;
};

QCUR_HD u128 u128_add(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1u : 0u);
  return r;
}

QCUR_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// (a * b) mod 2^128
QCUR_HD u128 u128_mul(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo * b.lo;
  r.hi = mulhi64(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
  return r;
}

// PCG_DEFAULT_MULTIPLIER_128
QCUR_HD u128 pcg_mult() { return u128{0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL}; }

struct Pcg64 {
  u128 state;
  u128 inc;  // always odd

  QCUR_HD void step() { state = u128_add(u128_mul(state, pcg_mult()), inc); }

  // XSL-RR output of the *advanced* state (numpy steps first, then outputs).
  QCUR_HD uint64_t next_u64() {
    step();
    uint64_t x = state.hi ^ state.lo;
    unsigned rot = (unsigned)(state.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }

  // Generator.random(): 53 random bits scaled by 2^-53.
  QCUR_HD double next_double() { return (double)(next_u64() >> 11) * (1.0 / 9007199254740992.0); }

  // Jump ahead by `delta` steps (Brown's LCG skip-ahead), as
  // numpy's bit_generator.advance(delta).
  QCUR_HD void advance(uint64_t delta) {
    u128 acc_mult{0, 1}, acc_plus{0, 0};
    u128 cur_mult = pcg_mult(), cur_plus = inc;
    while (delta > 0) {
      if (delta & 1u) {
        acc_mult = u128_mul(acc_mult, cur_mult);
        acc_plus = u128_add(u128_mul(acc_plus, cur_mult), cur_plus);
      }
      cur_plus = u128_mul(u128_add(cur_mult, u128{0, 1}), cur_plus);
      cur_mult = u128_mul(cur_mult, cur_mult);
      delta >>= 1;
    }
    state = u128_add(u128_mul(acc_mult, state), acc_plus);
  }
};

// numpy SeedSequence(entropy).generate_state(4, uint64) followed by
// PCG64's set_seed(state = words[0:2], inc = words[2:4]).
// `entropy` holds the seed as little-endian 32-bit words (seed 0 -> {0}).
QCUR_HD Pcg64 pcg64_from_entropy(const uint32_t* entropy, int nwords) {
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
  const uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) -> uint32_t {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    v ^= v >> 16;
    return v;
  };
  auto mix = [](uint32_t x, uint32_t y) -> uint32_t {
    uint32_t r = MIX_L * x - MIX_R * y;
    r ^= r >> 16;
    return r;
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < nwords ? entropy[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < nwords; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(entropy[s]));
  // generate_state(8 uint32 words) viewed as 4 little-endian uint64
  uint32_t hb = INIT_B;
  uint32_t w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  uint64_t s64[4];
  for (int i = 0; i < 4; ++i) s64[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  // pcg64_set_seed: initstate = (s64[0] << 64) | s64[1]; initseq = (s64[2] << 64) | s64[3]
  u128 initstate{s64[0], s64[1]};
  u128 initseq{s64[2], s64[3]};
  Pcg64 g;
  g.state = u128{0, 0};
  g.inc = u128{(initseq.hi << 1) | (initseq.lo >> 63), (initseq.lo << 1) | 1u};
  g.step();
  g.state = u128_add(g.state, initstate);
  g.step();
  return g;
}

}  // namespace qcur
