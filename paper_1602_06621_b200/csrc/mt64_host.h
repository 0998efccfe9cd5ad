// mt64_host.h -- MT19937-64 seeding and GF(2) jump polynomials (host side).
#pragma once

#include <cstdint>

namespace eqb {
namespace mt {

constexpr int kN = 312;        // state words
constexpr int kM = 156;        // middle offset
constexpr int kDegree = 19937; // degree of the characteristic polynomial
constexpr int kPolyWords = 312;  // ceil(19937 / 64)

uint64_t temper(uint64_t y);

// Raw mt19937_64 state after SeededRng(seed, stream) (src/rng.cpp:19-27):
// window W_0 = x[0..311]; output k is temper(x[312 + k]).
void seed_state(uint64_t seed, uint64_t stream, uint64_t out[kN]);

// x^(2^a) mod phi(x), bits 0..19936 in kPolyWords words.  Computed by repeated
// squaring the first time it is asked for, then cached for the process.
bool jump_poly_pow2(int a, uint64_t out[kPolyWords]);

// Host restatement of the device jump (for tests): out = sum_i r_i W_{p+i}.
void jump_window_host(const uint64_t win[kN], const uint64_t poly[kPolyWords],
                      uint64_t out[kN]);

}  // namespace mt
}  // namespace eqb
