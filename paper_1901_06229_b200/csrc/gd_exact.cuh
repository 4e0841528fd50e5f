// Exact FP64 device arithmetic: the reference's formulas with the reference's evaluation order and
// no FMA contraction (every op is an explicit _rn intrinsic, which nvcc never fuses). Results are
// bit-identical with the reference built without -march. Paths are relative to
// /root/reference/proj.
#pragma once

#include <cstdint>

#include "gd_internal.h"

namespace gdk {

struct V3d {
  double x, y, z;
};
struct Qd {
  double w, x, y, z;
};

__device__ __forceinline__ V3d vadd(V3d a, V3d b) {
  return {__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y), __dadd_rn(a.z, b.z)};
}
__device__ __forceinline__ V3d vsub(V3d a, V3d b) {
  return {__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)};
}
__device__ __forceinline__ V3d vscale(double s, V3d v) {  // operator*(double, Vec3), geometry.hpp:25
  return {__dmul_rn(s, v.x), __dmul_rn(s, v.y), __dmul_rn(s, v.z)};
}
__device__ __forceinline__ double vdot(V3d a, V3d b) {  // geometry.hpp:29
  return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}
__device__ __forceinline__ V3d vcross(V3d a, V3d b) {  // geometry.hpp:30-32
  return {__dsub_rn(__dmul_rn(a.y, b.z), __dmul_rn(a.z, b.y)),
          __dsub_rn(__dmul_rn(a.z, b.x), __dmul_rn(a.x, b.z)),
          __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}

// Rotation::apply (geometry.hpp:67-74): v + w t + q x t with t = 2 (q x v).
__device__ __forceinline__ V3d qapply(const Qd& q, V3d v) {
  const V3d qv{q.x, q.y, q.z};
  const V3d t = vscale(2.0, vcross(qv, v));
  return vadd(vadd(v, vscale(q.w, t)), vcross(qv, t));
}

// rotated_about (geometry.hpp:100-102).
__device__ __forceinline__ V3d rotated_about(V3d p, V3d c, const Qd& q) {
  return vadd(qapply(q, vsub(p, c)), c);
}

// Generic load: the field may be staged in shared memory (K1b) or read from global memory.
__device__ __forceinline__ double fld(const DevPocket& pk, uint32_t ix, uint32_t iy, uint32_t iz) {
  return pk.field[(size_t(iz) * pk.dims[1] + iy) * pk.dims[0] + ix];  // scoring.hpp:24-26
}

// sample_field (scoring.cpp:9-38).
__device__ __forceinline__ double sample_exact(const DevPocket& pk, V3d p) {
  const double gx = __ddiv_rn(__dsub_rn(p.x, pk.origin[0]), pk.spacing);
  const double gy = __ddiv_rn(__dsub_rn(p.y, pk.origin[1]), pk.spacing);
  const double gz = __ddiv_rn(__dsub_rn(p.z, pk.origin[2]), pk.spacing);
  if (gx < 0.0 || gy < 0.0 || gz < 0.0 || gx > pk.maxc[0] || gy > pk.maxc[1] || gz > pk.maxc[2]) {
    return 0.0;
  }
  uint32_t ix = uint32_t(__double2ull_rz(gx));
  uint32_t iy = uint32_t(__double2ull_rz(gy));
  uint32_t iz = uint32_t(__double2ull_rz(gz));
  if (ix > pk.dims[0] - 2) ix = pk.dims[0] - 2;
  if (iy > pk.dims[1] - 2) iy = pk.dims[1] - 2;
  if (iz > pk.dims[2] - 2) iz = pk.dims[2] - 2;
  const double fx = __dsub_rn(gx, double(ix));
  const double fy = __dsub_rn(gy, double(iy));
  const double fz = __dsub_rn(gz, double(iz));
  const double ux = __dsub_rn(1.0, fx), uy = __dsub_rn(1.0, fy), uz = __dsub_rn(1.0, fz);
  const double c00 = __dadd_rn(__dmul_rn(fld(pk, ix, iy, iz), ux), __dmul_rn(fld(pk, ix + 1, iy, iz), fx));
  const double c10 =
      __dadd_rn(__dmul_rn(fld(pk, ix, iy + 1, iz), ux), __dmul_rn(fld(pk, ix + 1, iy + 1, iz), fx));
  const double c01 =
      __dadd_rn(__dmul_rn(fld(pk, ix, iy, iz + 1), ux), __dmul_rn(fld(pk, ix + 1, iy, iz + 1), fx));
  const double c11 = __dadd_rn(__dmul_rn(fld(pk, ix, iy + 1, iz + 1), ux),
                               __dmul_rn(fld(pk, ix + 1, iy + 1, iz + 1), fx));
  const double c0 = __dadd_rn(__dmul_rn(c00, uy), __dmul_rn(c10, fy));
  const double c1 = __dadd_rn(__dmul_rn(c01, uy), __dmul_rn(c11, fy));
  return __dadd_rn(__dmul_rn(c0, uz), __dmul_rn(c1, fz));
}

// d^2 - thr^2 of a pair in bump_check's arithmetic (scoring.cpp:52-58): negative iff the pair clashes.
__device__ __forceinline__ double pair_margin_exact(V3d a, V3d b, double ra, double rb, double cf) {
  const V3d d = vsub(a, b);
  const double thr = __dmul_rn(cf, __dadd_rn(ra, rb));
  return __dsub_rn(vdot(d, d), __dmul_rn(thr, thr));
}

// Non-bonded pair clash test of bump_check (scoring.cpp:52-58): d^2 < (cf (ra + rb))^2.
__device__ __forceinline__ bool pair_clash_exact(V3d a, V3d b, double ra, double rb, double cf) {
  const V3d d = vsub(a, b);
  const double thr = __dmul_rn(cf, __dadd_rn(ra, rb));
  return vdot(d, d) < __dmul_rn(thr, thr);
}

}  // namespace gdk
