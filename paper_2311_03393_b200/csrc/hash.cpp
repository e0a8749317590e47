// Count-sketch hash pair (h, s) — PAPER.md §3.1 P:L200-204 ("two pair-wise independent hash
// functions h: [d]->[k] and s: [d]->{-1,+1}", selected at random from their families).
// Reading 2: Carter–Wegman 2-universal family over the Mersenne prime
// p = 2^61 - 1, keyed by the stream id (so §3.3 add/delete never moves another stream), its
// parameters (a, b, c, e) drawn from splitmix64(seed).  Host code; 128-bit products.
#include <stdint.h>

#include "internal.h"

namespace skmp {

static const uint64_t kP61 = (uint64_t(1) << 61) - 1;

static inline uint64_t splitmix_next(uint64_t& state) {
  state += 0x9E3779B97F4A7C15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// (x mod p) for x < 2^122 via the Mersenne identity 2^61 = 1 (mod p).
static inline uint64_t mod_p61(unsigned __int128 x) {
  uint64_t lo = (uint64_t)(x & kP61);
  uint64_t hi = (uint64_t)(x >> 61);
  uint64_t r = lo + (hi & kP61) + (uint64_t)(hi >> 61);
  r = (r & kP61) + (r >> 61);
  if (r >= kP61) r -= kP61;
  return r;
}

void cw_params(uint64_t seed, uint64_t* a, uint64_t* b, uint64_t* c, uint64_t* e) {
  uint64_t st = seed;
  do { *a = splitmix_next(st) % kP61; } while (*a == 0);
  *b = splitmix_next(st) % kP61;
  do { *c = splitmix_next(st) % kP61; } while (*c == 0);
  *e = splitmix_next(st) % kP61;
}

void hash_plan(const uint64_t* ids, int64_t d, int32_t k, uint64_t seed, int32_t* g, int8_t* s) {
  uint64_t a, b, c, e;
  cw_params(seed, &a, &b, &c, &e);
  for (int64_t j = 0; j < d; ++j) {
    uint64_t x = ids[j] % kP61;
    uint64_t hg = mod_p61((unsigned __int128)a * x + b);
    uint64_t hs = mod_p61((unsigned __int128)c * x + e);
    if (g) g[j] = (int32_t)(hg % (uint64_t)k);
    if (s) s[j] = (hs & 1) ? -1 : 1;
  }
}

}  // namespace skmp
