// gen.cpp -- seeded synthetic instances for BASELINE.json's configs
// (libequil_gen.so; bench/test input only, not part of the hot path).
//
// The reference's own generator (src/experiments.cpp:80-122) keeps a dense
// m*n bitmap and caps m*n <= 2^28, so it cannot produce configs 3-5; these
// generators are written from the config text instead.
// Every row draws from its own counter-seeded stream, so the output does not
// depend on the thread count.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace {

struct Rng {  // splitmix64 stream
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double uniform() { return (static_cast<double>(next() >> 11) + 0.5) * 0x1.0p-53; }
  double normal() {  // Box-Muller, one value per call
    const double u1 = uniform(), u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
  uint64_t below(uint64_t n) { return next() % n; }
};

uint64_t stream_seed(uint64_t seed, uint64_t stream, uint64_t idx) {
  Rng r(seed * 0x9E3779B97F4A7C15ULL ^ (stream + 1) * 0xD1B54A32D192ED03ULL);
  r.s ^= idx * 0xA24BAED4963EE407ULL;
  r.next();
  return r.next();
}

template <class F>
void parallel_for(int64_t n, F&& f) {
  const int T = std::max(1u, std::thread::hardware_concurrency());
  const int64_t chunk = (n + T - 1) / T;
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) {
    const int64_t b = t * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    th.emplace_back([=, &f] {
      for (int64_t i = b; i < e; ++i) f(i);
    });
  }
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

// Row lengths. kind 0: fixed p0; kind 1: truncated Zipf(exponent p0) on
// [1, p1]; kind 2: round(LogNormal(mu = p0, sigma = p1)) clamped to [1, n].
// Writes row_ptr (m + 1 entries), returns nnz.
int64_t gen_row_ptr(int64_t m, int64_t n, int kind, double p0, double p1, uint64_t seed,
                    int64_t* row_ptr) {
  std::vector<double> cdf;
  if (kind == 1) {
    const int64_t kmax = static_cast<int64_t>(p1);
    cdf.resize(kmax);
    double acc = 0.0;
    for (int64_t k = 1; k <= kmax; ++k) cdf[k - 1] = (acc += std::pow(static_cast<double>(k), -p0));
    for (auto& c : cdf) c /= acc;
  }
  std::vector<int64_t> len(m);
  parallel_for(m, [&](int64_t i) {
    Rng r(stream_seed(seed, 0, i));
    int64_t l = 0;
    if (kind == 0) {
      l = static_cast<int64_t>(p0);
    } else if (kind == 1) {
      const double u = r.uniform();
      l = (std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin()) + 1;
    } else {
      l = std::llround(std::exp(p0 + p1 * r.normal()));
    }
    len[i] = std::max<int64_t>(1, std::min<int64_t>(l, n));
  });
  row_ptr[0] = 0;
  for (int64_t i = 0; i < m; ++i) row_ptr[i + 1] = row_ptr[i] + len[i];
  return row_ptr[m];
}

// Distinct uniform columns per row (sorted) and values
// N(0,1) * exp(sr * N(0,1))_row * exp(sc * N(0,1))_col.
void gen_fill(int64_t m, int64_t n, const int64_t* row_ptr, uint64_t seed, double sr,
              double sc, int32_t* col, double* val) {
  std::vector<double> cs(n), rs(m);
  parallel_for(n, [&](int64_t j) {
    Rng r(stream_seed(seed, 2, j));
    cs[j] = std::exp(sc * r.normal());
  });
  parallel_for(m, [&](int64_t i) {
    Rng r(stream_seed(seed, 1, i));
    rs[i] = std::exp(sr * r.normal());
  });
  parallel_for(m, [&](int64_t i) {
    Rng r(stream_seed(seed, 3, i));
    const int64_t b = row_ptr[i], L = row_ptr[i + 1] - b;
    int32_t* c = col + b;
    if (L * 2 > n) {  // dense-ish row: choose by selection sampling
      int64_t need = L;
      int64_t k = 0;
      for (int64_t j = 0; j < n && need > 0; ++j)
        if (r.below(n - j) < static_cast<uint64_t>(need)) {
          c[k++] = static_cast<int32_t>(j);
          --need;
        }
    } else {
      int64_t have = 0;
      while (have < L) {
        for (int64_t k = have; k < L; ++k) c[k] = static_cast<int32_t>(r.below(n));
        std::sort(c, c + L);
        have = std::unique(c, c + L) - c;
      }
    }
    for (int64_t k = 0; k < L; ++k) val[b + k] = (r.normal() * rs[i]) * cs[c[k]];
  });
}

void gen_dense(int64_t m, int64_t n, uint64_t seed, double sr, double sc, double* a) {
  std::vector<double> cs(n), rs(m);
  parallel_for(n, [&](int64_t j) {
    Rng r(stream_seed(seed, 2, j));
    cs[j] = std::exp(sc * r.normal());
  });
  parallel_for(m, [&](int64_t i) {
    Rng r(stream_seed(seed, 1, i));
    rs[i] = std::exp(sr * r.normal());
  });
  parallel_for(m, [&](int64_t i) {
    Rng r(stream_seed(seed, 3, i));
    for (int64_t j = 0; j < n; ++j) a[i * n + j] = (r.normal() * rs[i]) * cs[j];
  });
}

void gen_normal(uint64_t seed, uint64_t stream, int64_t count, double* out) {
  parallel_for((count + 4095) / 4096, [&](int64_t blk) {
    Rng r(stream_seed(seed, 10 + stream, blk));
    const int64_t b = blk * 4096, e = std::min(count, b + 4096);
    for (int64_t k = b; k < e; ++k) out[k] = r.normal();
  });
}

}  // extern "C"
