// Host-side FP64 pieces of the reference that need libm (sin/cos) and therefore stay on the host so
// that their bits equal the reference's: the rotation grid, the dihedral (cos, sin) table and the
// per-restart starting transform. This translation unit family is compiled with
// -ffp-contract=off and without -march. Paths relative to /root/reference/proj.
#pragma once

#include <cmath>
#include <cstdint>
#include <string_view>

namespace gdh {

constexpr double kPi = 3.14159265358979323846;  // geometry.hpp:10
constexpr double kTwoPi = 2.0 * kPi;            // geometry.hpp:11

struct SplitMix64 {  // prng.hpp:11-31
  uint64_t state;
  explicit SplitMix64(uint64_t s) : state(s) {}
  uint64_t next() {
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + uniform() * (hi - lo); }
  uint64_t below(uint64_t n) { return n > 0 ? next() % n : 0; }
};

inline uint64_t fnv1a64(std::string_view text) {  // prng.hpp:33-40
  uint64_t h = 0xCBF29CE484222325ull;
  for (char c : text) {
    h ^= static_cast<unsigned char>(c);
    h *= 0x100000001B3ull;
  }
  return h;
}

inline uint64_t mix_seed(uint64_t a, uint64_t b) {  // prng.hpp:43-46
  SplitMix64 g(a ^ (b + 0x9E3779B97F4A7C15ull + (a << 6) + (a >> 2)));
  return g.next();
}

struct Q {
  double w, x, y, z;
};

inline Q about_axis(double ax, double ay, double az, double angle) {  // geometry.hpp:46-50
  const double half = 0.5 * angle;
  const double s = std::sin(half);
  return {std::cos(half), ax * s, ay * s, az * s};
}

inline Q compose(const Q& a, const Q& o) {  // geometry.hpp:56-61
  return {a.w * o.w - a.x * o.x - a.y * o.y - a.z * o.z, a.w * o.x + a.x * o.w + a.y * o.z - a.z * o.y,
          a.w * o.y - a.x * o.z + a.y * o.w + a.z * o.x, a.w * o.z + a.x * o.y - a.y * o.x + a.z * o.w};
}

inline Q from_euler_zyz(double alpha, double beta, double gamma) {  // geometry.cpp:9-14
  return compose(compose(about_axis(0.0, 0.0, 1.0, alpha), about_axis(0.0, 1.0, 0.0, beta)),
                 about_axis(0.0, 0.0, 1.0, gamma));
}

inline Q random_rotation(SplitMix64& rng) {  // docking.cpp:19-30 (Shoemake)
  const double u1 = rng.uniform();
  const double u2 = rng.uniform();
  const double u3 = rng.uniform();
  const double r1 = std::sqrt(1.0 - u1);
  const double r2 = std::sqrt(u1);
  Q q{r2 * std::cos(kTwoPi * u3), r1 * std::sin(kTwoPi * u2), r1 * std::cos(kTwoPi * u2),
      r2 * std::sin(kTwoPi * u3)};
  const double n = std::sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
  return {q.w / n, q.x / n, q.y / n, q.z / n};
}

}  // namespace gdh
