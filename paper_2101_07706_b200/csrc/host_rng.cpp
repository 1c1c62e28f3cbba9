// Host-side RNG runtime: the reference's stream derivation and batch selection, native.
//
// The reference derives every random stream with
//   spawn_rng(seed, *labels) = default_rng(SeedSequence([seed & 2^64-1] + sha256_words(repr(l))...))
// (seeding.py:17-27) and picks each worker's batch with
//   spawn_rng(seed, "batch", epoch, it, w).choice(worker_train, take, replace=False)
// (training.py:488-491).  Doing that through numpy costs ~0.35 ms per worker-iteration
// on the host, more than the whole GPU iteration, so it is restated here bit-exactly:
// SHA-256, numpy's SeedSequence pool mixing + generate_state, PCG64 seeding
// (pcg64_set_seed), next_uint64/next_uint32 buffering, Lemire bounded integers and
// both branches of Generator.choice(replace=False) (Floyd's hash-set / tail shuffle).
// Every output is checked against numpy in tests/test_host_rng.py.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>

#include "skg_internal.h"

namespace skg {

// ---------------------------------------------------------------- SHA-256 (FIPS 180-4)
namespace {
const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

inline uint32_t rotr32(uint32_t x, int r) { return (x >> r) | (x << (32 - r)); }

void sha256(const uint8_t* msg, size_t len, uint8_t out[32]) {
  uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                   0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  std::vector<uint8_t> buf(msg, msg + len);
  uint64_t bits = (uint64_t)len * 8;
  buf.push_back(0x80);
  while (buf.size() % 64 != 56) buf.push_back(0);
  for (int i = 7; i >= 0; --i) buf.push_back((uint8_t)(bits >> (8 * i)));
  for (size_t off = 0; off < buf.size(); off += 64) {
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = (uint32_t)buf[off + 4 * i] << 24 | (uint32_t)buf[off + 4 * i + 1] << 16 |
             (uint32_t)buf[off + 4 * i + 2] << 8 | (uint32_t)buf[off + 4 * i + 3];
    for (int i = 16; i < 64; ++i) {
      uint32_t s0 = rotr32(w[i - 15], 7) ^ rotr32(w[i - 15], 18) ^ (w[i - 15] >> 3);
      uint32_t s1 = rotr32(w[i - 2], 17) ^ rotr32(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; ++i) {
      uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
      uint32_t ch = (e & f) ^ (~e & g);
      uint32_t t1 = hh + S1 + ch + K256[i] + w[i];
      uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
      uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
      uint32_t t2 = S0 + mj;
      hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
  }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) out[4 * i + j] = (uint8_t)(h[i] >> (24 - 8 * j));
}

// ---------------------------------------------------------------- numpy SeedSequence
const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu,
               MULT_B = 0x58f38dedu, MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;

void seedseq_generate_u64x4(const std::vector<uint32_t>& ent, uint64_t out[4]) {
  uint32_t pool[4];
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    v ^= v >> 16;
    return v;
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    r ^= r >> 16;
    return r;
  };
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < (int)ent.size() ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (size_t s = 4; s < ent.size(); ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));
  uint32_t hb = INIT_B, st[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> 16;
    st[i] = v;
  }
  for (int i = 0; i < 4; ++i) out[i] = (uint64_t)st[2 * i] | ((uint64_t)st[2 * i + 1] << 32);
}
}  // namespace

// ---------------------------------------------------------------- PCG64 (numpy flavour)
static inline u128 mk128(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }
const u128 PCG_MULT = mk128(0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL);

uint64_t Pcg64::next64() {
  state = state * PCG_MULT + inc;
  uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
  unsigned r = (unsigned)(state >> 122);
  return (x >> r) | (x << ((64 - r) & 63));
}

uint32_t Pcg64::next32() {
  if (has32) {
    has32 = 0;
    return u32;
  }
  uint64_t v = next64();
  has32 = 1;
  u32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

// numpy random_bounded_uint64(bitgen, 0, rng, 0, use_masked=false)
uint64_t Pcg64::bounded(uint64_t rng) {
  if (rng == 0) return 0;
  if (rng <= 0xFFFFFFFFULL) {
    if (rng == 0xFFFFFFFFULL) return next32();
    uint32_t r32 = (uint32_t)rng, excl = r32 + 1;
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      uint32_t thr = (0xFFFFFFFFu - r32) % excl;
      while (left < thr) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return m >> 32;
  }
  if (rng == ~0ULL) return next64();
  uint64_t excl = rng + 1;
  u128 m = (u128)next64() * excl;
  uint64_t left = (uint64_t)m;
  if (left < excl) {
    uint64_t thr = (~0ULL - rng) % excl;
    while (left < thr) {
      m = (u128)next64() * excl;
      left = (uint64_t)m;
    }
  }
  return (uint64_t)(m >> 64);
}

Pcg64 pcg64_from_seedseq(const uint64_t s[4]) {
  // pcg64_set_seed: PCG_128BIT_CONSTANT(seed[0], seed[1]) i.e. seed[0] is the high word
  u128 initstate = mk128(s[0], s[1]);
  u128 initseq = mk128(s[2], s[3]);
  Pcg64 g;
  g.inc = (initseq << 1) | 1;
  g.state = 0;
  g.state = g.state * PCG_MULT + g.inc;
  g.state += initstate;
  g.state = g.state * PCG_MULT + g.inc;
  g.has32 = 0;
  g.u32 = 0;
  return g;
}

Pcg64 spawn_pcg64(uint64_t master_seed, const std::vector<std::string>& label_reprs) {
  std::vector<uint32_t> ent;
  // _int_to_uint32_array(master & 2^64-1): little-endian 32-bit words, at least one
  uint64_t m = master_seed;
  if (m == 0) ent.push_back(0);
  while (m) {
    ent.push_back((uint32_t)m);
    m >>= 32;
  }
  for (const auto& rep : label_reprs) {
    uint8_t dig[32];
    sha256(reinterpret_cast<const uint8_t*>(rep.data()), rep.size(), dig);
    for (int o = 0; o < 16; o += 4)
      ent.push_back((uint32_t)dig[o] | (uint32_t)dig[o + 1] << 8 | (uint32_t)dig[o + 2] << 16 |
                    (uint32_t)dig[o + 3] << 24);
  }
  uint64_t st[4];
  seedseq_generate_u64x4(ent, st);
  return pcg64_from_seedseq(st);
}

// Generator.choice(pop, size, replace=False, p=None, shuffle=True) index set (unsorted).
void choice_without_replacement(Pcg64& g, int64_t pop, int64_t size, int64_t* out) {
  if (size <= 0) return;
  const int64_t cutoff = 50;  // shuffle=True
  if (pop > 10000 && size > pop / cutoff) {
    std::vector<int64_t> idx(pop);
    for (int64_t i = 0; i < pop; ++i) idx[i] = i;
    int64_t first = std::max<int64_t>(pop - size, 1);
    for (int64_t i = pop - 1; i >= first; --i) {
      int64_t j = (int64_t)g.bounded((uint64_t)i);
      std::swap(idx[i], idx[j]);
    }
    std::memcpy(out, idx.data() + (pop - size), sizeof(int64_t) * size);
    return;
  }
  uint64_t set_size = (uint64_t)(1.2 * (double)size);
  uint64_t mask = set_size;
  mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
  mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
  std::vector<uint64_t> hs(mask + 1, ~0ULL);
  for (int64_t j = pop - size; j < pop; ++j) {
    uint64_t val = g.bounded((uint64_t)j);
    uint64_t loc = val & mask;
    while (hs[loc] != ~0ULL && hs[loc] != val) loc = (loc + 1) & mask;
    if (hs[loc] == ~0ULL) {
      hs[loc] = val;
      out[j - pop + size] = (int64_t)val;
    } else {
      loc = (uint64_t)j & mask;
      while (hs[loc] != ~0ULL) loc = (loc + 1) & mask;
      hs[loc] = (uint64_t)j;
      out[j - pop + size] = j;
    }
  }
  // the trailing _shuffle_int only permutes the (later sorted) result
}

std::string repr_str(const char* s) { return std::string("'") + s + "'"; }
std::string repr_int(int64_t v) { return std::to_string(v); }

}  // namespace skg
