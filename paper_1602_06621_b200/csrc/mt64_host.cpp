// mt64_host.cpp -- host half of the device MT19937-64 sign stream (K1).
//
// The reference draws probe signs from std::mt19937_64 seeded through
// splitmix64 (src/rng.cpp:9-36, stream 17 = include/equil/streams.hpp:17), in
// the order n signs for s then m signs for w per iteration
// (src/estimator.cpp:6 via src/equilibrate.cpp:165-166).  The stream never
// depends on the iterate, so all T*(n+m) signs are produced up front by
// independent device segments.  Segment g starts at output g*L; its 312-word
// window is reached by GF(2) jump-ahead: W_{p+J} = sum_i r_i W_{p+i} with
// r(x) = x^J mod phi(x), phi the characteristic polynomial of the MT19937-64
// transition (degree 19937), recovered here once per process by
// Berlekamp-Massey on the generator's own output bits.
#include "mt64_host.h"

#include <cstring>
#include <mutex>
#include <vector>

namespace eqb {
namespace mt {

namespace {

constexpr uint64_t kA = 0xB5026F5AA96619E9ULL;
constexpr uint64_t kUM = 0xFFFFFFFF80000000ULL;
constexpr uint64_t kLM = 0x000000007FFFFFFFULL;

uint64_t splitmix64(uint64_t& state) {
  state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

using Poly = std::vector<uint64_t>;  // bit i = coefficient of x^i

inline int getbit(const Poly& p, size_t i) { return (p[i >> 6] >> (i & 63)) & 1; }
inline void flipbit(Poly& p, size_t i) { p[i >> 6] ^= 1ULL << (i & 63); }

// p ^= q << s (bitwise shift), p sized large enough
void xor_shifted(Poly& p, const Poly& q, size_t s) {
  const size_t ws = s >> 6, bs = s & 63;
  for (size_t w = 0; w < q.size(); ++w) {
    if (!q[w]) continue;
    p[w + ws] ^= q[w] << bs;
    if (bs && w + ws + 1 < p.size()) p[w + ws + 1] ^= q[w] >> (64 - bs);
  }
}

struct CharPoly {
  Poly phi;                    // degree kDegree, 313 words
  std::vector<Poly> shifted;   // phi << s for s in [0, 64), 314 words each
};

CharPoly* build_charpoly() {
  // Output-bit sequence (MSB of each tempered output) of an arbitrary seed.
  const size_t N = 2 * kDegree + 64;
  std::vector<uint8_t> s(N);
  {
    uint64_t st[kN];
    seed_state(12345, 0, st);
    std::vector<uint64_t> x(st, st + kN);
    x.reserve(N + kN + 1);
    for (size_t k = 0; k < N; ++k) {
      const uint64_t y = (x[k] & kUM) | (x[k + 1] & kLM);
      uint64_t nw = x[k + kM] ^ (y >> 1) ^ ((y & 1) ? kA : 0);
      x.push_back(nw);
      s[k] = static_cast<uint8_t>(temper(nw) >> 63);
    }
  }
  // Berlekamp-Massey over GF(2).  Connection poly C: s_k = sum_{i>=1} C_i s_{k-i}.
  const size_t W = (N + 63) / 64 + 2;
  // reversed sequence bits: rv bit (N-1-k) = s_k, so the window s_{k-L..k}
  // maps to a contiguous, ascending bit range of rv starting at N-1-k.
  Poly rv(W, 0);
  for (size_t k = 0; k < N; ++k)
    if (s[k]) flipbit(rv, N - 1 - k);
  Poly Cp(W, 0), Bp(W, 0), Tp;
  Cp[0] = Bp[0] = 1;
  size_t L = 0, mshift = 1;
  for (size_t k = 0; k < N; ++k) {
    // discrepancy d = sum_{i=0..L} C_i s_{k-i}: bit i of C against rv bit (N-1-k+i)
    const size_t off = N - 1 - k;
    const size_t ow = off >> 6, ob = off & 63;
    uint64_t acc = 0;
    const size_t nw = (L >> 6) + 1;
    for (size_t w = 0; w < nw; ++w) {
      uint64_t r = rv[w + ow] >> ob;
      if (ob && w + ow + 1 < W) r |= rv[w + ow + 1] << (64 - ob);
      uint64_t c = Cp[w];
      if (w == nw - 1 && ((L + 1) & 63)) c &= (1ULL << ((L + 1) & 63)) - 1;
      acc ^= c & r;
    }
    const int d = __builtin_parityll(acc);
    if (!d) {
      ++mshift;
    } else if (2 * L <= k) {
      Tp = Cp;
      xor_shifted(Cp, Bp, mshift);
      L = k + 1 - L;
      Bp.swap(Tp);
      mshift = 1;
    } else {
      xor_shifted(Cp, Bp, mshift);
      ++mshift;
    }
  }
  if (L != static_cast<size_t>(kDegree)) return nullptr;
  auto* cp = new CharPoly;
  cp->phi.assign(kPolyWords + 1, 0);
  for (size_t i = 0; i <= L; ++i)  // phi_i = C_{L-i}
    if (getbit(Cp, L - i)) flipbit(cp->phi, i);
  cp->shifted.resize(64);
  for (int sft = 0; sft < 64; ++sft) {
    cp->shifted[sft].assign(kPolyWords + 2, 0);
    xor_shifted(cp->shifted[sft], cp->phi, sft);
  }
  return cp;
}

std::once_flag g_once;
CharPoly* g_cp = nullptr;
std::mutex g_mu;
std::vector<Poly> g_pow2;  // g_pow2[a] = x^(2^a) mod phi

const CharPoly& charpoly() {
  std::call_once(g_once, [] { g_cp = build_charpoly(); });
  return *g_cp;
}

// p (degree < 2*kDegree) reduced mod phi, result kPolyWords words
Poly reduce(Poly p) {
  const CharPoly& cp = charpoly();
  for (size_t b = 2 * kDegree; b-- > static_cast<size_t>(kDegree);) {
    if (!getbit(p, b)) continue;
    const size_t s = b - kDegree;
    const Poly& q = cp.shifted[s & 63];
    const size_t ws = s >> 6;
    for (size_t w = 0; w < q.size() && w + ws < p.size(); ++w) p[w + ws] ^= q[w];
  }
  p.resize(kPolyWords);
  return p;
}

Poly square_mod(const Poly& a) {
  Poly p(2 * kPolyWords + 2, 0);
  for (size_t i = 0; i < static_cast<size_t>(kDegree); ++i)
    if (getbit(a, i)) flipbit(p, 2 * i);
  return reduce(std::move(p));
}

}  // namespace

uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

void seed_state(uint64_t seed, uint64_t stream, uint64_t out[kN]) {
  // SeededRng::SeededRng (src/rng.cpp:19-27), then mt19937_64::seed.
  uint64_t state = seed;
  uint64_t mixed = splitmix64(state);
  state ^= stream * 0xD1B54A32D192ED03ULL + 0x2545F4914F6CDD1DULL;
  mixed ^= splitmix64(state);
  out[0] = mixed;
  for (int i = 1; i < kN; ++i)
    out[i] = 6364136223846793005ULL * (out[i - 1] ^ (out[i - 1] >> 62)) +
             static_cast<uint64_t>(i);
}

bool jump_poly_pow2(int a, uint64_t out[kPolyWords]) {
  if (a < 0 || a > 62) return false;
  const CharPoly& cp = charpoly();
  if (!g_cp) return false;
  (void)cp;
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_pow2.empty()) {
    Poly x(kPolyWords, 0);
    x[0] = 2;  // x^1
    g_pow2.push_back(x);
  }
  while (static_cast<int>(g_pow2.size()) <= a) g_pow2.push_back(square_mod(g_pow2.back()));
  std::memcpy(out, g_pow2[a].data(), kPolyWords * sizeof(uint64_t));
  return true;
}

void jump_window_host(const uint64_t win[kN], const uint64_t poly[kPolyWords],
                      uint64_t out[kN]) {
  std::vector<uint64_t> x(win, win + kN);
  const size_t need = kDegree + kN;
  x.reserve(need + 1);
  for (size_t k = 0; x.size() < need; ++k) {
    const uint64_t y = (x[k] & kUM) | (x[k + 1] & kLM);
    x.push_back(x[k + kM] ^ (y >> 1) ^ ((y & 1) ? kA : 0));
  }
  for (int j = 0; j < kN; ++j) out[j] = 0;
  for (size_t i = 0; i < static_cast<size_t>(kDegree); ++i) {
    if (!((poly[i >> 6] >> (i & 63)) & 1)) continue;
    for (int j = 0; j < kN; ++j) out[j] ^= x[i + j];
  }
}

}  // namespace mt
}  // namespace eqb
