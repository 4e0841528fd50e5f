/* TEST INFRASTRUCTURE — NOT PRODUCT CODE. See geodock_oracle.h for the parity-pinning story.
 *
 * A scalar, single-threaded, FP64 restatement of the reference algorithm. Every function cites the
 * reference file:line (relative to /root/reference/proj) whose arithmetic it restates. Evaluation
 * order is kept identical (left-associative sums, no FMA contraction: built with
 * -ffp-contract=off) so results are bit-identical with the reference on the same libm.
 */
#include "geodock_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define K_PI 3.14159265358979323846 /* geometry.hpp:10 */
static const double kTwoPi = 2.0 * K_PI; /* geometry.hpp:11 */

static char g_err[512];
const char* go_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- prng.hpp:11-46 */
typedef struct { uint64_t state; } sm64;

static uint64_t sm_next(sm64* g) { /* prng.hpp:16-21 */
  uint64_t z = (g->state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double sm_uniform(sm64* g) { return (double)(sm_next(g) >> 11) * 0x1.0p-53; } /* :24 */
static double sm_uniform_in(sm64* g, double lo, double hi) { return lo + sm_uniform(g) * (hi - lo); }
static uint64_t sm_below(sm64* g, uint64_t n) { return n > 0 ? sm_next(g) % n : 0; } /* :30 */

uint64_t go_splitmix_next(uint64_t* state) {
  sm64 g = {*state};
  uint64_t v = sm_next(&g);
  *state = g.state;
  return v;
}

uint64_t go_fnv1a64(const char* s, uint64_t len) { /* prng.hpp:33-40 */
  uint64_t h = 0xCBF29CE484222325ull;
  for (uint64_t i = 0; i < len; ++i) {
    h ^= (unsigned char)s[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

uint64_t go_mix_seed(uint64_t a, uint64_t b) { /* prng.hpp:43-46 */
  sm64 g = {a ^ (b + 0x9E3779B97F4A7C15ull + (a << 6) + (a >> 2))};
  return sm_next(&g);
}

/* ---------------------------------------------------------------- geometry.hpp:17-102 */
typedef struct { double x, y, z; } v3;
typedef struct { double w, x, y, z; } quat;

static v3 v_add(v3 a, v3 b) { v3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static v3 v_sub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static v3 v_scale(double s, v3 v) { v3 r = {s * v.x, s * v.y, s * v.z}; return r; }
static double v_dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 v_cross(v3 a, v3 b) {
  v3 r = {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
  return r;
}

static quat q_about_axis(v3 axis, double angle) { /* geometry.hpp:46-50 */
  const double half = 0.5 * angle;
  const double s = sin(half);
  quat q = {cos(half), axis.x * s, axis.y * s, axis.z * s};
  return q;
}

static quat q_compose(quat a, quat o) { /* geometry.hpp:56-61 */
  quat r = {a.w * o.w - a.x * o.x - a.y * o.y - a.z * o.z,
            a.w * o.x + a.x * o.w + a.y * o.z - a.z * o.y,
            a.w * o.y - a.x * o.z + a.y * o.w + a.z * o.x,
            a.w * o.z + a.x * o.y - a.y * o.x + a.z * o.w};
  return r;
}

static v3 q_apply(quat q, v3 v) { /* geometry.hpp:67-74: v + w t + q x t, t = 2 q x v */
  const v3 qv = {q.x, q.y, q.z};
  const v3 t = v_scale(2.0, v_cross(qv, v));
  return v_add(v_add(v, v_scale(q.w, t)), v_cross(qv, t));
}

static v3 rotated_about(v3 p, v3 c, quat r) { return v_add(q_apply(r, v_sub(p, c)), c); } /* :100-102 */

static v3 centroid(const v3* p, uint32_t n) { /* geometry.cpp:40-46 */
  v3 s = {0.0, 0.0, 0.0};
  for (uint32_t i = 0; i < n; ++i) s = v_add(s, p[i]);
  return v_scale(1.0 / (double)n, s);
}

static quat from_euler_zyz(double a, double b, double g) { /* geometry.cpp:9-14 */
  const v3 z = {0.0, 0.0, 1.0}, y = {0.0, 1.0, 0.0};
  return q_compose(q_compose(q_about_axis(z, a), q_about_axis(y, b)), q_about_axis(z, g));
}

static quat* make_grid(const uint32_t st[3], uint64_t* size) { /* geometry.cpp:16-34 */
  const uint64_t n = (uint64_t)st[0] * st[1] * st[2];
  quat* q = (quat*)malloc(sizeof(quat) * (n ? n : 1));
  uint64_t at = 0;
  for (unsigned i = 0; i < st[0]; ++i) {
    const double alpha = kTwoPi * (double)i / (double)st[0];
    for (unsigned j = 0; j < st[1]; ++j) {
      const double beta = st[1] == 1 ? 0.0 : K_PI * (double)j / (double)(st[1] - 1);
      for (unsigned k = 0; k < st[2]; ++k) {
        const double gamma = kTwoPi * (double)k / (double)st[2];
        q[at++] = from_euler_zyz(alpha, beta, gamma);
      }
    }
  }
  *size = n;
  return q;
}

int go_rotation_grid(const uint32_t steps[3], double* q_out) {
  if (!steps[0] || !steps[1] || !steps[2]) {
    snprintf(g_err, sizeof g_err, "rotation grid steps must all be >= 1");
    return 3;
  }
  uint64_t n;
  quat* q = make_grid(steps, &n);
  for (uint64_t i = 0; i < n; ++i) {
    q_out[4 * i] = q[i].w;
    q_out[4 * i + 1] = q[i].x;
    q_out[4 * i + 2] = q[i].y;
    q_out[4 * i + 3] = q[i].z;
  }
  free(q);
  return 0;
}

/* ---------------------------------------------------------------- scoring.hpp:18-37, scoring.cpp */
typedef struct {
  v3 origin;
  double spacing;
  uint64_t dims[3];
  const double* field;
} pocket;

static double at3(const pocket* p, uint64_t ix, uint64_t iy, uint64_t iz) {
  return p->field[(iz * p->dims[1] + iy) * p->dims[0] + ix]; /* scoring.hpp:24-26 */
}

static double sample_field(const pocket* pk, v3 p) { /* scoring.cpp:9-38 */
  const double gx = (p.x - pk->origin.x) / pk->spacing;
  const double gy = (p.y - pk->origin.y) / pk->spacing;
  const double gz = (p.z - pk->origin.z) / pk->spacing;
  const double mx = (double)(pk->dims[0] - 1);
  const double my = (double)(pk->dims[1] - 1);
  const double mz = (double)(pk->dims[2] - 1);
  if (gx < 0.0 || gy < 0.0 || gz < 0.0 || gx > mx || gy > my || gz > mz) return 0.0;
  uint64_t ix = (uint64_t)gx, iy = (uint64_t)gy, iz = (uint64_t)gz;
  if (ix > pk->dims[0] - 2) ix = pk->dims[0] - 2;
  if (iy > pk->dims[1] - 2) iy = pk->dims[1] - 2;
  if (iz > pk->dims[2] - 2) iz = pk->dims[2] - 2;
  const double fx = gx - (double)ix, fy = gy - (double)iy, fz = gz - (double)iz;
  const double c00 = at3(pk, ix, iy, iz) * (1.0 - fx) + at3(pk, ix + 1, iy, iz) * fx;
  const double c10 = at3(pk, ix, iy + 1, iz) * (1.0 - fx) + at3(pk, ix + 1, iy + 1, iz) * fx;
  const double c01 = at3(pk, ix, iy, iz + 1) * (1.0 - fx) + at3(pk, ix + 1, iy, iz + 1) * fx;
  const double c11 = at3(pk, ix, iy + 1, iz + 1) * (1.0 - fx) + at3(pk, ix + 1, iy + 1, iz + 1) * fx;
  const double c0 = c00 * (1.0 - fy) + c10 * fy;
  const double c1 = c01 * (1.0 - fy) + c11 * fy;
  return c0 * (1.0 - fz) + c1 * fz;
}

int go_sample_field(const uint32_t dims[3], const double origin[3], double spacing,
                    const double* field, uint64_t n, const double* pts, double* out) {
  pocket pk = {{origin[0], origin[1], origin[2]}, spacing, {dims[0], dims[1], dims[2]}, field};
  for (uint64_t i = 0; i < n; ++i) {
    v3 p = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    out[i] = sample_field(&pk, p);
  }
  return 0;
}

/* ---------------------------------------------------------------- molecule (finalized ligand) */
typedef struct {
  uint32_t n, nb, nr;
  const char* name;
  uint32_t name_len;
  v3* pos;                 /* current pose */
  const double* radius;
  unsigned char* adj;      /* n*n, molecule.cpp:80-86 */
  uint32_t* rot_i;
  uint32_t* rot_j;
  uint32_t** moving;       /* per rotamer, sorted (molecule.cpp:88-98) */
  uint32_t* moving_len;
  double* dih;
} ligand;

static double score_pose(const ligand* L, const pocket* pk) { /* scoring.cpp:40-45 */
  double sum = 0.0;
  for (uint32_t a = 0; a < L->n; ++a) sum += sample_field(pk, L->pos[a]);
  return sum / (double)L->n;
}

static int bump_check(const ligand* L, const v3* pos, double cf) { /* scoring.cpp:47-61 */
  for (uint32_t a = 0; a + 1 < L->n; ++a) {
    for (uint32_t b = a + 1; b < L->n; ++b) {
      if (L->adj[(size_t)a * L->n + b]) continue;
      const v3 d = v_sub(pos[a], pos[b]);
      const double thr = cf * (L->radius[a] + L->radius[b]);
      if (v_dot(d, d) < thr * thr) return 0;
    }
  }
  return 1;
}

/* rotate_fragment (molecule.cpp:145-174) writing into out (a copy of pos). Returns 0 or 4 (degenerate). */
static int rotate_fragment(const ligand* L, const v3* pos, uint32_t r, double angle, v3* out,
                           double* dih_out) {
  memcpy(out, pos, sizeof(v3) * L->n);
  *dih_out = L->dih[r];
  if (angle == 0.0) return 0;
  const v3 pi = pos[L->rot_i[r]], pj = pos[L->rot_j[r]];
  const v3 delta = v_sub(pj, pi);
  const double len = sqrt(v_dot(delta, delta));
  if (len < 1e-12) {
    snprintf(g_err, sizeof g_err, "rotamer axis atoms coincide in ligand '%.*s'", (int)L->name_len, L->name);
    return 4;
  }
  const v3 axis = v_scale(1.0 / len, delta);
  const quat q = q_about_axis(axis, angle);
  for (uint32_t m = 0; m < L->moving_len[r]; ++m) {
    const uint32_t a = L->moving[r][m];
    if (a == L->rot_j[r]) continue;
    out[a] = rotated_about(pos[a], pi, q);
  }
  double d = fmod(L->dih[r] + angle, kTwoPi);
  if (d < 0.0) d += kTwoPi;
  *dih_out = d;
  return 0;
}

/* ---------------------------------------------------------------- generate.cpp */
int go_make_pocket(const uint32_t dims[3], double spacing, const double origin[3], uint32_t blobs,
                   uint64_t seed, double* field) { /* generate.cpp:27-66 */
  sm64 rng = {go_mix_seed(seed, go_fnv1a64("pocket", 6))};
  const v3 lo = {origin[0], origin[1], origin[2]};
  const v3 hi = {origin[0] + spacing * (double)(dims[0] - 1), origin[1] + spacing * (double)(dims[1] - 1),
                 origin[2] + spacing * (double)(dims[2] - 1)};
  v3* cen = (v3*)malloc(sizeof(v3) * (blobs ? blobs : 1));
  double* inv = (double*)malloc(sizeof(double) * (blobs ? blobs : 1));
  double* amp = (double*)malloc(sizeof(double) * (blobs ? blobs : 1));
  for (uint32_t b = 0; b < blobs; ++b) {
    cen[b].x = sm_uniform_in(&rng, lo.x, hi.x);
    cen[b].y = sm_uniform_in(&rng, lo.y, hi.y);
    cen[b].z = sm_uniform_in(&rng, lo.z, hi.z);
    const double sigma = sm_uniform_in(&rng, 2.0, 5.0);
    inv[b] = 1.0 / (2.0 * sigma * sigma);
    amp[b] = sm_uniform_in(&rng, 0.4, 1.0);
  }
  for (uint64_t iz = 0; iz < dims[2]; ++iz)
    for (uint64_t iy = 0; iy < dims[1]; ++iy)
      for (uint64_t ix = 0; ix < dims[0]; ++ix) {
        const v3 g = {(double)ix, (double)iy, (double)iz};
        const v3 p = v_add(lo, v_scale(spacing, g));
        double v = 0.0;
        for (uint32_t b = 0; b < blobs; ++b) {
          const v3 d = v_sub(p, cen[b]);
          v += amp[b] * exp(-v_dot(d, d) * inv[b]);
        }
        field[(iz * dims[1] + iy) * dims[0] + ix] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
      }
  free(cen);
  free(inv);
  free(amp);
  return 0;
}

static v3 random_unit_vector(sm64* rng) { /* generate.cpp:13-23 (Marsaglia) */
  for (;;) {
    const double u = sm_uniform_in(rng, -1.0, 1.0);
    const double v = sm_uniform_in(rng, -1.0, 1.0);
    const double s = u * u + v * v;
    if (s >= 1.0 || s == 0.0) continue;
    const double f = 2.0 * sqrt(1.0 - s);
    v3 r = {u * f, v * f, 1.0 - 2.0 * s};
    return r;
  }
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y);
}

int go_make_library(uint64_t count, uint64_t atoms, uint64_t rotamers, uint64_t seed, double* xyz,
                    double* radius, uint32_t* bonds, uint32_t* rots) { /* generate.cpp:68-109 */
  const uint64_t n = atoms < 1 ? 1 : atoms;
  const uint64_t nr = rotamers < n - 1 ? rotamers : n - 1;
  const uint64_t lig_seed = go_mix_seed(seed, go_fnv1a64("ligand", 6));
  v3* p = (v3*)malloc(sizeof(v3) * n);
  uint64_t* edge = (uint64_t*)malloc(sizeof(uint64_t) * (n > 1 ? n - 1 : 1));
  uint32_t* par = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (uint64_t index = 0; index < count; ++index) {
    sm64 rng = {go_mix_seed(lig_seed, index)};
    double* rad = radius + index * n;
    p[0].x = p[0].y = p[0].z = 0.0;
    rad[0] = sm_uniform_in(&rng, 0.6, 0.9);
    for (uint64_t t = 1; t < n; ++t) {
      const uint64_t parent = sm_below(&rng, t);
      const v3 dir = random_unit_vector(&rng);
      p[t] = v_add(p[parent], v_scale(1.5, dir));
      rad[t] = sm_uniform_in(&rng, 0.6, 0.9);
      par[t] = (uint32_t)parent;
    }
    const uint64_t E = n - 1;
    for (uint64_t e = 0; e < E; ++e) edge[e] = e;
    for (uint64_t e = 0; e + 1 < E; ++e) {
      const uint64_t sw = e + sm_below(&rng, E - e);
      const uint64_t tmp = edge[e];
      edge[e] = edge[sw];
      edge[sw] = tmp;
    }
    const uint64_t keep = nr < E ? nr : E;
    qsort(edge, keep, sizeof(uint64_t), cmp_u64);
    for (uint64_t a = 0; a < n; ++a) {
      xyz[3 * (index * n + a)] = p[a].x;
      xyz[3 * (index * n + a) + 1] = p[a].y;
      xyz[3 * (index * n + a) + 2] = p[a].z;
    }
    for (uint64_t e = 0; e < E; ++e) { /* bond e = (parent(e+1), e+1) */
      bonds[2 * (index * E + e)] = par[e + 1];
      bonds[2 * (index * E + e) + 1] = (uint32_t)(e + 1);
    }
    for (uint64_t r = 0; r < keep; ++r) {
      rots[2 * (index * keep + r)] = par[edge[r] + 1];
      rots[2 * (index * keep + r) + 1] = (uint32_t)(edge[r] + 1);
    }
  }
  free(p);
  free(edge);
  free(par);
  return 0;
}

/* ---------------------------------------------------------------- ligand construction */
/* finalize_ligand (molecule.cpp:80-99): adjacency + moving set = component of atom_j after
 * deleting edge (i, j). Validation (molecule.cpp:176-238) is reduced to what the dock needs:
 * indices in range, connected graph, rotamer bond present and splitting the graph. */
static int build_ligand(ligand* L, uint32_t l, const uint32_t* atom_off, const double* xyz,
                        const double* radius, const uint32_t* bond_off, const uint32_t* bonds,
                        const uint32_t* rot_off, const uint32_t* rots, const double* dihedrals,
                        const uint32_t* name_off, const char* names) {
  memset(L, 0, sizeof *L);
  L->n = atom_off[l + 1] - atom_off[l];
  L->nb = bond_off[l + 1] - bond_off[l];
  L->nr = rot_off[l + 1] - rot_off[l];
  L->name = names + name_off[l];
  L->name_len = name_off[l + 1] - name_off[l];
  if (L->n == 0) {
    snprintf(g_err, sizeof g_err, "ligand has no atoms");
    return 2;
  }
  const uint32_t n = L->n;
  L->pos = (v3*)malloc(sizeof(v3) * n);
  for (uint32_t a = 0; a < n; ++a) {
    const size_t g = (size_t)atom_off[l] + a;
    L->pos[a].x = xyz[3 * g];
    L->pos[a].y = xyz[3 * g + 1];
    L->pos[a].z = xyz[3 * g + 2];
  }
  L->radius = radius + atom_off[l];
  L->adj = (unsigned char*)calloc((size_t)n * n, 1);
  uint32_t* deg = (uint32_t*)calloc(n, sizeof(uint32_t));
  for (uint32_t b = 0; b < L->nb; ++b) {
    const uint32_t u = bonds[2 * (bond_off[l] + b)], v = bonds[2 * (bond_off[l] + b) + 1];
    if (u >= n || v >= n || u == v) {
      free(deg);
      snprintf(g_err, sizeof g_err, "bond index out of range or self-bond");
      return 2;
    }
    L->adj[(size_t)u * n + v] = L->adj[(size_t)v * n + u] = 1;
  }
  free(deg);
  L->rot_i = (uint32_t*)malloc(sizeof(uint32_t) * (L->nr + 1));
  L->rot_j = (uint32_t*)malloc(sizeof(uint32_t) * (L->nr + 1));
  L->dih = (double*)malloc(sizeof(double) * (L->nr + 1));
  L->moving = (uint32_t**)calloc(L->nr + 1, sizeof(uint32_t*));
  L->moving_len = (uint32_t*)calloc(L->nr + 1, sizeof(uint32_t));
  unsigned char* seen = (unsigned char*)malloc(n);
  uint32_t* stack = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
  /* connectivity from atom 0 */
  memset(seen, 0, n);
  uint32_t sp = 0, cnt = 1;
  stack[sp++] = 0;
  seen[0] = 1;
  while (sp) {
    const uint32_t u = stack[--sp];
    for (uint32_t v = 0; v < n; ++v)
      if (L->adj[(size_t)u * n + v] && !seen[v]) {
        seen[v] = 1;
        ++cnt;
        stack[sp++] = v;
      }
  }
  int rc = 0;
  if (cnt != n) {
    snprintf(g_err, sizeof g_err, "bond graph is not connected");
    rc = 2;
  }
  for (uint32_t r = 0; r < L->nr && rc == 0; ++r) {
    const uint32_t i = rots[2 * (rot_off[l] + r)], j = rots[2 * (rot_off[l] + r) + 1];
    L->rot_i[r] = i;
    L->rot_j[r] = j;
    L->dih[r] = dihedrals ? dihedrals[rot_off[l] + r] : 0.0;
    if (i >= n || j >= n || !L->adj[(size_t)i * n + j]) {
      snprintf(g_err, sizeof g_err, "rotamer %u is not a bond", r);
      rc = 2;
      break;
    }
    memset(seen, 0, n);
    sp = 0;
    stack[sp++] = j;
    seen[j] = 1;
    while (sp) {
      const uint32_t u = stack[--sp];
      for (uint32_t v = 0; v < n; ++v) {
        if (!L->adj[(size_t)u * n + v]) continue;
        if ((u == i && v == j) || (u == j && v == i)) continue;
        if (!seen[v]) {
          seen[v] = 1;
          stack[sp++] = v;
        }
      }
    }
    if (seen[i]) {
      snprintf(g_err, sizeof g_err, "rotamer bond (%u,%u) does not disconnect graph", i, j);
      rc = 2;
      break;
    }
    L->moving[r] = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (uint32_t a = 0; a < n; ++a)
      if (seen[a]) L->moving[r][L->moving_len[r]++] = a;
  }
  free(seen);
  free(stack);
  return rc;
}

static void free_ligand(ligand* L) {
  free(L->pos);
  free(L->adj);
  for (uint32_t r = 0; r < L->nr; ++r) free(L->moving ? L->moving[r] : NULL);
  free(L->moving);
  free(L->moving_len);
  free(L->rot_i);
  free(L->rot_j);
  free(L->dih);
}

/* ---------------------------------------------------------------- docking.cpp */
static quat random_rotation(sm64* rng) { /* docking.cpp:19-30 (Shoemake) */
  const double u1 = sm_uniform(rng), u2 = sm_uniform(rng), u3 = sm_uniform(rng);
  const double r1 = sqrt(1.0 - u1), r2 = sqrt(u1);
  quat q = {r2 * cos(kTwoPi * u3), r1 * sin(kTwoPi * u2), r1 * cos(kTwoPi * u2), r2 * sin(kTwoPi * u3)};
  const double nrm = sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
  quat o = {q.w / nrm, q.x / nrm, q.y / nrm, q.z / nrm};
  return o;
}

/* generate_starting_pose (docking.cpp:52-69) into start[]. */
static void starting_pose(const ligand* L, const v3* base, unsigned pose_id, uint64_t seed,
                          const pocket* pk, v3* start) {
  sm64 rng = {go_mix_seed(go_mix_seed(seed, go_fnv1a64(L->name, L->name_len)), pose_id)};
  const quat r = random_rotation(&rng);
  const v3 lo = pk->origin;
  const v3 hi = {pk->origin.x + pk->spacing * (double)(pk->dims[0] - 1),
                 pk->origin.y + pk->spacing * (double)(pk->dims[1] - 1),
                 pk->origin.z + pk->spacing * (double)(pk->dims[2] - 1)};
  v3 target;
  target.x = sm_uniform_in(&rng, lo.x, hi.x);
  target.y = sm_uniform_in(&rng, lo.y, hi.y);
  target.z = sm_uniform_in(&rng, lo.z, hi.z);
  const v3 c = centroid(base, L->n);
  for (uint32_t a = 0; a < L->n; ++a) start[a] = v_add(q_apply(r, v_sub(base[a], c)), target);
}

int go_dock_library(uint32_t n_lig, const uint32_t* atom_off, const double* xyz,
                    const double* radius, const uint32_t* bond_off, const uint32_t* bonds,
                    const uint32_t* rot_off, const uint32_t* rots, const double* dihedrals,
                    const uint32_t* name_off, const char* names, const uint32_t dims[3],
                    const double origin[3], double spacing, const double* field,
                    uint32_t n_restarts, uint32_t reps, const uint32_t steps[3],
                    uint32_t dihedral_steps, double clash, uint64_t seed, double* best_score,
                    uint32_t* best_restart, uint64_t* score_calls, double* phase,
                    double* final_xyz, double* final_dih, uint32_t* align_index,
                    double* align_score, double* restart_score, int32_t* step_k,
                    double* step_score) {
  if (!(clash > 0.0) || clash > 1.0) {
    snprintf(g_err, sizeof g_err, "clash_factor must lie in (0, 1]");
    return 3;
  }
  if (!steps[0] || !steps[1] || !steps[2]) {
    snprintf(g_err, sizeof g_err, "rotation grid steps must all be >= 1");
    return 3;
  }
  pocket pk = {{origin[0], origin[1], origin[2]}, spacing, {dims[0], dims[1], dims[2]}, field};
  uint64_t G;
  quat* grid = make_grid(steps, &G);
  const double delta = kTwoPi / (double)dihedral_steps; /* docking.cpp:129 */
  int rc = 0;
  for (uint32_t l = 0; l < n_lig && rc == 0; ++l) {
    ligand L;
    rc = build_ligand(&L, l, atom_off, xyz, radius, bond_off, bonds, rot_off, rots, dihedrals,
                      name_off, names);
    if (rc) {
      free_ligand(&L);
      break;
    }
    const uint32_t n = L.n, R = L.nr;
    v3* base = (v3*)malloc(sizeof(v3) * n);
    memcpy(base, L.pos, sizeof(v3) * n);
    v3* start = (v3*)malloc(sizeof(v3) * n);
    v3* pose = (v3*)malloc(sizeof(v3) * n);
    v3* cand = (v3*)malloc(sizeof(v3) * n);
    v3* bestc = (v3*)malloc(sizeof(v3) * n);
    v3* best_pose = (v3*)malloc(sizeof(v3) * n);
    double* base_dih = (double*)malloc(sizeof(double) * (R + 1));
    double* best_dih = (double*)malloc(sizeof(double) * (R + 1));
    memcpy(base_dih, L.dih, sizeof(double) * R);
    double best = 0.0;
    int have = 0;
    unsigned best_id = 0;
    for (unsigned pid = 0; pid < n_restarts && rc == 0; ++pid) {
      const size_t p = (size_t)l * n_restarts + pid;
      /* align_restarts (docking.cpp:178-195) */
      starting_pose(&L, base, pid, seed, &pk, start);
      const v3 c = centroid(start, n); /* best_rotation_in_range (docking.cpp:71-91) */
      uint64_t bidx = (uint64_t)-1;
      double bscore = -1.0;
      for (uint64_t g = 0; g < G; ++g) {
        double sum = 0.0;
        for (uint32_t a = 0; a < n; ++a) sum += sample_field(&pk, rotated_about(start[a], c, grid[g]));
        const double s = sum / (double)n;
        if (s > bscore || bidx == (uint64_t)-1) {
          bidx = g;
          bscore = s;
        }
      }
      /* apply_rotation_choice (docking.cpp:110-118) */
      const v3 c2 = centroid(start, n);
      for (uint32_t a = 0; a < n; ++a) pose[a] = rotated_about(start[a], c2, grid[bidx]);
      double score = bscore;
      memcpy(L.dih, base_dih, sizeof(double) * R);
      if (align_index) align_index[p] = (uint32_t)bidx;
      if (align_score) align_score[p] = bscore;
      /* finish_dock (docking.cpp:197-235) + optimize_pass (:155-167) + dihedral_step (:127-149) */
      for (unsigned rep = 0; rep < reps && rc == 0; ++rep) {
        for (uint32_t r = 0; r < R && rc == 0; ++r) {
          int committed = 0;
          unsigned bk = 0;
          double bs = 0.0, bdih = 0.0;
          for (unsigned k = 0; k < dihedral_steps; ++k) {
            double dk;
            rc = rotate_fragment(&L, pose, r, k == 0 ? 0.0 : delta * (double)k, cand, &dk);
            if (rc) break;
            const ligand* Lc = &L;
            const v3* keep = L.pos;
            L.pos = cand;
            const double s = score_pose(Lc, &pk);
            L.pos = (v3*)keep;
            const int eligible = bump_check(&L, cand, clash);
            if (eligible && (!committed || s > bs)) {
              committed = 1;
              bk = k;
              bs = s;
              bdih = dk;
              memcpy(bestc, cand, sizeof(v3) * n);
            }
          }
          if (rc) break;
          if (committed) {
            memcpy(pose, bestc, sizeof(v3) * n);
            L.dih[r] = bdih;
            score = bs;
          }
          const size_t si = (size_t)rot_off[l] * n_restarts * reps + ((size_t)pid * reps + rep) * R + r;
          if (step_k) step_k[si] = committed ? (int32_t)bk : -1;
          if (step_score) step_score[si] = score;
        }
      }
      if (restart_score) restart_score[p] = score;
      if (!have || score > best) {
        have = 1;
        best = score;
        best_id = pid;
        memcpy(best_pose, pose, sizeof(v3) * n);
        memcpy(best_dih, L.dih, sizeof(double) * R);
      }
    }
    if (rc == 0) {
      best_score[l] = best;
      best_restart[l] = best_id;
      const uint64_t align_calls = (uint64_t)n_restarts * G;
      const uint64_t opt_calls = (uint64_t)n_restarts * reps * R * dihedral_steps;
      score_calls[l] = align_calls + opt_calls; /* docking.cpp:226 (recorded == closed form :44-50) */
      phase[2 * l] = (double)align_calls * 1e-7; /* docking.hpp:27, docking.cpp:227-229 */
      phase[2 * l + 1] = (double)opt_calls * 1e-7;
      for (uint32_t a = 0; a < n; ++a) {
        final_xyz[3 * ((size_t)atom_off[l] + a)] = best_pose[a].x;
        final_xyz[3 * ((size_t)atom_off[l] + a) + 1] = best_pose[a].y;
        final_xyz[3 * ((size_t)atom_off[l] + a) + 2] = best_pose[a].z;
      }
      for (uint32_t r = 0; r < R; ++r) final_dih[rot_off[l] + r] = best_dih[r];
    }
    free(base);
    free(start);
    free(pose);
    free(cand);
    free(bestc);
    free(best_pose);
    free(base_dih);
    free(best_dih);
    free_ligand(&L);
  }
  free(grid);
  return rc;
}
