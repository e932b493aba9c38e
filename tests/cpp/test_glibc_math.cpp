// Host check of csrc/glibc_math.cuh against the live glibc log/cos -- TEST ONLY.
// Inputs are the RngStream::normal domain (rng.hpp:111-116): u1 = 1 - k 2^-53
// and x = fl(2 pi k 2^-53), plus the region boundaries of __cos_fma.
#define __host__
#define __device__
#define __forceinline__ inline
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "glibc_math.cuh"

static uint64_t sm(uint64_t& s) {  // splitmix64
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static bool same(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 4000000;
  uint64_t s = 12345;
  long bad_log = 0, bad_cos = 0, bad_norm = 0;
  for (long i = 0; i < n; ++i) {
    uint64_t k = sm(s) >> 11;
    if ((i & 7) == 0) k &= (1ull << (49 + (i >> 3) % 4)) - 1;  // bias toward u1 near 1
    const double u1 = 1.0 - double(k) * 0x1.0p-53;
    if (!same(fnb::glibc::log(u1), std::log(u1))) { if (bad_log++ < 5) printf("log mismatch %a\n", u1); }
    uint64_t k2 = sm(s) >> 11;
    if ((i & 15) == 1) k2 &= (1ull << (30 + (i >> 4) % 20)) - 1;  // small arguments
    const double x = 6.283185307179586476925286766559 * (double(k2) * 0x1.0p-53);
    if (!same(fnb::glibc::cos(x), std::cos(x))) { if (bad_cos++ < 5) printf("cos mismatch %a\n", x); }
    const double u0 = double(k) * 0x1.0p-53, uu = double(k2) * 0x1.0p-53;
    const double want = 0.3 + (1.7 * std::sqrt(-2.0 * std::log(1.0 - u0))) * std::cos(6.283185307179586476925286766559 * uu);
    if (!same(fnb::glibc::normal_from_uniforms(u0, uu, 0.3, 1.7), want)) bad_norm++;
  }
  // boundaries of the __cos_fma regions and multiples of pi/2
  const double edges[] = {0x1p-27, 0.855469, 2.426265, 1.5707963267948966, 3.141592653589793, 4.71238898038469,
                          6.283185307179586, 0.126, 1.5707963267948966 - 0.126, 1.5707963267948966 + 0.126};
  for (double e : edges)
    for (int d = -20000; d <= 20000; ++d) {
      const double x = e + d * 0x1p-40;
      if (x < 0 || x >= 6.283185307179586) continue;
      if (!same(fnb::glibc::cos(x), std::cos(x))) { if (bad_cos++ < 10) printf("cos edge mismatch %a\n", x); }
    }
  printf("samples %ld  log mismatches %ld  cos mismatches %ld  normal mismatches %ld\n", n, bad_log, bad_cos, bad_norm);
  return (bad_log || bad_cos || bad_norm) ? 1 : 0;
}
