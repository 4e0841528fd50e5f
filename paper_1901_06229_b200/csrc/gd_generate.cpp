// Synthetic workload generator (generate.hpp:12-31, generate.cpp:13-109 in /root/reference/proj):
// the pocket (Gaussian blobs) and the random tree-shaped ligand library that BASELINE.json's
// configs are defined through. Same PRNG streams and FP64 arithmetic as the reference
// (compiled with -ffp-contract=off, no -march), so the GPU and the oracles see identical inputs;
// tests/test_host.py checks it bit-for-bit against the reference build.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "gd_host_math.h"
#include "geodock_b200.h"

namespace {

struct V {
  double x, y, z;
};

V random_unit_vector(gdh::SplitMix64& rng) {  // generate.cpp:13-23 (Marsaglia)
  while (true) {
    const double u = rng.uniform(-1.0, 1.0);
    const double v = rng.uniform(-1.0, 1.0);
    const double s = u * u + v * v;
    if (s >= 1.0 || s == 0.0) continue;
    const double f = 2.0 * std::sqrt(1.0 - s);
    return {u * f, v * f, 1.0 - 2.0 * s};
  }
}

}  // namespace

extern "C" {

int gd_make_pocket(const uint32_t dims[3], double spacing, const double origin[3], uint32_t blobs,
                   uint64_t seed, double* field) {  // generate.cpp:27-66
  if (!dims || !origin || !field) return GD_ERR_ARGUMENT;
  gdh::SplitMix64 rng(gdh::mix_seed(seed, gdh::fnv1a64("pocket")));
  const V lo{origin[0], origin[1], origin[2]};
  const V hi{origin[0] + spacing * static_cast<double>(dims[0] - 1),
             origin[1] + spacing * static_cast<double>(dims[1] - 1),
             origin[2] + spacing * static_cast<double>(dims[2] - 1)};
  struct Blob {
    V c;
    double inv, amp;
  };
  std::vector<Blob> bl;
  for (uint32_t b = 0; b < blobs; ++b) {
    Blob x;
    x.c.x = rng.uniform(lo.x, hi.x);
    x.c.y = rng.uniform(lo.y, hi.y);
    x.c.z = rng.uniform(lo.z, hi.z);
    const double sigma = rng.uniform(2.0, 5.0);
    x.inv = 1.0 / (2.0 * sigma * sigma);
    x.amp = rng.uniform(0.4, 1.0);
    bl.push_back(x);
  }
  for (size_t iz = 0; iz < dims[2]; ++iz)
    for (size_t iy = 0; iy < dims[1]; ++iy)
      for (size_t ix = 0; ix < dims[0]; ++ix) {
        const V p{origin[0] + spacing * static_cast<double>(ix), origin[1] + spacing * static_cast<double>(iy),
                  origin[2] + spacing * static_cast<double>(iz)};
        double v = 0.0;
        for (const Blob& b : bl) {
          const V d{p.x - b.c.x, p.y - b.c.y, p.z - b.c.z};
          v += b.amp * std::exp(-(d.x * d.x + d.y * d.y + d.z * d.z) * b.inv);
        }
        field[(iz * dims[1] + iy) * dims[0] + ix] = std::clamp(v, 0.0, 1.0);
      }
  return GD_OK;
}

int gd_make_library_range(uint64_t first, uint64_t count, uint64_t atoms, uint64_t rotamers, uint64_t seed,
                          double* xyz, double* radius, uint32_t* bonds, uint32_t* rots) {  // generate.cpp:68-109
  if ((count && (!xyz || !radius)) || (!bonds && atoms > 1)) return GD_ERR_ARGUMENT;
  const uint64_t n = std::max<uint64_t>(1, atoms);
  const uint64_t nr = std::min<uint64_t>(rotamers, n - 1);
  const uint64_t E = n - 1;
  const uint64_t lig_seed = gdh::mix_seed(seed, gdh::fnv1a64("ligand"));
  // every ligand draws from its own stream mix_seed(lig_seed, index) (generate.cpp:76): a range of
  // the library is generated directly, and blocks of ligands go to all host threads
  auto block = [&](uint64_t i0, uint64_t i1) {
    std::vector<V> p(n);
    std::vector<uint64_t> parent(n, 0), edge(E);
    for (uint64_t i = i0; i < i1; ++i) {
      const uint64_t index = first + i;
      gdh::SplitMix64 rng(gdh::mix_seed(lig_seed, index));
      double* rad = radius + i * n;
      p[0] = {0.0, 0.0, 0.0};
      rad[0] = rng.uniform(0.6, 0.9);
      for (uint64_t t = 1; t < n; ++t) {
        const uint64_t par = rng.below(t);
        const V d = random_unit_vector(rng);
        p[t] = {p[par].x + 1.5 * d.x, p[par].y + 1.5 * d.y, p[par].z + 1.5 * d.z};
        rad[t] = rng.uniform(0.6, 0.9);
        parent[t] = par;
      }
      for (uint64_t e = 0; e < E; ++e) edge[e] = e;
      for (uint64_t e = 0; e + 1 < E; ++e) std::swap(edge[e], edge[e + rng.below(E - e)]);
      const uint64_t keep = std::min(nr, E);
      std::sort(edge.begin(), edge.begin() + keep);
      for (uint64_t a = 0; a < n; ++a) {
        xyz[3 * (i * n + a)] = p[a].x;
        xyz[3 * (i * n + a) + 1] = p[a].y;
        xyz[3 * (i * n + a) + 2] = p[a].z;
      }
      for (uint64_t e = 0; e < E; ++e) {
        bonds[2 * (i * E + e)] = uint32_t(parent[e + 1]);
        bonds[2 * (i * E + e) + 1] = uint32_t(e + 1);
      }
      for (uint64_t r = 0; r < keep; ++r) {
        rots[2 * (i * keep + r)] = uint32_t(parent[edge[r] + 1]);
        rots[2 * (i * keep + r) + 1] = uint32_t(edge[r] + 1);
      }
    }
  };
  const uint64_t hw = std::max(1u, std::thread::hardware_concurrency());
  const uint64_t nt = std::min<uint64_t>(hw, count / 2048 + 1);
  if (nt <= 1) {
    block(0, count);
    return GD_OK;
  }
  std::vector<std::thread> th;
  for (uint64_t t = 0; t < nt; ++t) th.emplace_back(block, count * t / nt, count * (t + 1) / nt);
  for (auto& t : th) t.join();
  return GD_OK;
}

int gd_make_library(uint64_t count, uint64_t atoms, uint64_t rotamers, uint64_t seed, double* xyz,
                    double* radius, uint32_t* bonds, uint32_t* rots) {
  return gd_make_library_range(0, count, atoms, rotamers, seed, xyz, radius, bonds, rots);
}

}  // extern "C"
