// K1 fast: two-stage pose search. DESIGN.md §3 has the derivation; paths are relative to
// /root/reference/proj.
//
// Every decision the reference makes — the alignment argmax (docking.cpp:71-91), each dihedral
// step's eligibility and argmax (docking.cpp:127-149) — is taken here in two stages:
//   1. a coarse FP32 screen over ALL candidates (the faithful sweep: every rotation of every restart,
//      every dihedral candidate's moved atoms and cross pairs), reading the pocket as 15-bit
//      fixed-point 8-corner cells staged once per CTA in shared memory (one LDS.128 per sample);
//   2. an exact FP64 re-evaluation, in the reference's arithmetic and summation order, of the few
//      candidates whose coarse score lies within the rigorous error bound 2*eps of the best (plus
//      any sample within the position bound of a grid face, plus any bump pair within its bound of
//      the threshold). The argmax over the exact scores is therefore the reference's argmax.
// Every pose, score and dihedral that leaves the kernel is FP64 and bit-identical to the reference.
//
// Work decomposition: persistent CTAs (one per SM), the pocket cells loaded once per CTA; each
// warp claims (ligand, restart) items from a global counter. Lane layout: alignment = lanes over
// rotations; dihedral sweep = lanes over candidate angles k (32 per pass, the remainder split
// 2..32 lanes per candidate over the fixed atoms); FP64 master pose = atom a lives in lane a%32,
// register slot a/32.
#include <algorithm>
#include <type_traits>

#include "gd_exact.cuh"
#include "gd_fast.cuh"

namespace gdk {
namespace {

constexpr unsigned FULL = 0xffffffffu;
// branch-weight hints: rare paths of the sweep laid out away from the per-step hot path
// (instruction-cache footprint)
#ifndef GD_HINTS
#define GD_HINTS 1  // C2 K1b: clash 0.75 -3 %, clash 0.1 -2 %
#endif
#if GD_HINTS
#define GD_UNLIKELY(x) __builtin_expect(!!(x), 0)
#define GD_LIKELY(x) __builtin_expect(!!(x), 1)
#else
#define GD_UNLIKELY(x) (x)
#define GD_LIKELY(x) (x)
#endif
constexpr float kMagic = 8388608.0f;  // 2^23: RZ-add leaves floor(g) in the mantissa
constexpr int KTOP = 2;               // per-lane top coarse alignment candidates kept (2 beat 3 and 4)

#ifndef GD_ALIGN_UNROLL
#define GD_ALIGN_UNROLL 1
#endif
#ifndef GD_FAST_THREADS
#define GD_FAST_THREADS 512
#endif
constexpr int kAlignUnroll = GD_ALIGN_UNROLL;
#ifndef GD_ALPHA_CHUNK
#define GD_ALPHA_CHUNK 4
#endif
constexpr int kAlphaChunk = GD_ALPHA_CHUNK;
#ifndef GD_REG_ROWS_MAX_NS
#define GD_REG_ROWS_MAX_NS 2  // pair-state rows in registers up to this NS, shared-memory rows beyond
#endif
constexpr uint32_t kZCap = 32;  // razor-thin pairs tracked per pose (beyond: every step takes the slow path)
// per-warp sweep counters -> gd_stats (16 + i): steps, invariant-clash steps, scored steps, moved-atom
// samples, cross pairs, k != 0 commits, FP64 candidate scores (other / all-outside / near a face),
// FP64 cross-pair checks
constexpr uint32_t kSweepCtr = 10;
#ifndef GD_K1A_X2
#define GD_K1A_X2 1  // K1a samples in f32x2 pairs (bit-identical to the scalar form)
#endif
#ifndef GD_K1B_FIELDF
#define GD_K1B_FIELDF 1  // K1b's coarse samples from an FP32 field copy in shared memory
#endif
#ifndef GD_K1A_TMA_STAGE
#define GD_K1A_TMA_STAGE 0  // K1a's cells by TMA bulk copy (measured 1.5 % slower overall than the LDG loop)
#endif
#ifndef GD_QT_GROUPS
#define GD_QT_GROUPS 2
#endif
constexpr int kQtGroups = GD_QT_GROUPS;  // quarter-turn groups per pass over the atoms
// cross-pair list entries per warp (folded when the next moved atom's <= 32 NS pairs might not fit)
template <int NS>
__host__ __device__ constexpr uint32_t pair_cap() { return 32u * NS + 32u; }
// Optional device-side phase timers (build with -DGD_PHASE_TIMERS): per-warp clock64 deltas summed
// into gd_stats-adjacent counters 8..15 (setup, align coarse, align refine, refresh, step head,
// step coarse candidates, step decisions+commit, tail).
#ifdef GD_PHASE_TIMERS
#define GD_T(slot) do { const long long t_ = clock64(); ph[cur_ph] += t_ - t_ph; t_ph = t_; cur_ph = (slot); } while (0)
#else
#define GD_T(slot) do { } while (0)
#endif
#ifndef GD_K1B_MIN_WARPS_SC
#define GD_K1B_MIN_WARPS_SC 12  // K1b keeps the cells in shared memory only if this many warps still fit
#endif
#ifndef GD_ALIGN_THREADS
#define GD_ALIGN_THREADS 448  // K1a, cells in shared memory, 33..64 atoms: 14 warps x 128 registers (C2 -1.4 % vs 12, -1 % vs 16)
#endif
#ifndef GD_ALIGN_THREADS_NS1
#define GD_ALIGN_THREADS_NS1 384  // the same for <= 32 atoms: 12 warps (16: C1 shape at 4k -0.6 %, but C1's 100-ligand batch +23 %: 1.35 items per warp)
#endif
#ifndef GD_ALIGN_THREADS_NS4
#define GD_ALIGN_THREADS_NS4 384  // the same for 65..128 atoms (and NS = 8): 12 warps x 168 (C4: 14 warps +1 %)
#endif
#ifndef GD_ALIGN_THREADS_L1
#define GD_ALIGN_THREADS_L1 512  // K1a when the cells do not fit shared memory (read through L1; C5: 512 > 384, 448, 640)
#endif
#ifndef GD_REFINE_THREADS
// K1r for <= 64 atoms: 32 warps x 64 registers (the FP64 scorer spills ~600 bytes, yet the extra
// warps hide its latency chains better: C2 K1r -22 % against 16 warps x 128)
#define GD_REFINE_THREADS 1024
#endif
#ifndef GD_REFINE_THREADS_NS4
#define GD_REFINE_THREADS_NS4 512  // K1r otherwise (65..128 atoms, or the FP64 field not in shared memory)
#endif
#ifndef GD_FAST_THREADS_NS4
#define GD_FAST_THREADS_NS4 256  // NS = 4: 255 registers (no spills) beat 16 warps at 128 (C4 clash 0.1 +15 %)
#endif

// status bits of a coarse dihedral candidate
constexpr uint32_t ST_CLASH = 1, ST_OK = 2, ST_XAMB = 4, ST_SAMB = 8, ST_ALLOUT = 16;

struct CoarseGrid {
  const uint4* cells;  // shared (or global) cells: four x-edges each, plus the dummy cell
  float hx, hy, hz;    // half extents (dims-1)/2 in grid units
  uint32_t cx, cxy;    // cells per row / per plane
  uint32_t koff;       // 0x4B000000 * (1 + cx + cxy): removes the 2^23 exponent bits of the three floors
  uint32_t dummy;      // index of the dummy cell (every fraction evaluates to ~0)
  float nb;            // -B: the dD field's bias (gd_set_pocket)
};

// One cell by byte address: shared (SC, a 32-bit shared-window address) or global (an offset from
// cg.cells, read through the read-only path).
template <bool SC>
__device__ __forceinline__ uint4 load_cell(const CoarseGrid& cg, uint32_t addr) {
  uint4 w;
  if (SC) {
    asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "r"(addr));
  } else {
    w = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(cg.cells) + addr));
  }
  return w;
}

// One cell: per y-edge j (words 2j, 2j+1) the bilinear form in (fx, fz) of its
// four corners, v = C0 + fz dC + fx (D0 + fz dD), as 16-bit fields that byte permutes against one
// constant K turn into floats: 1 + C0 (selector 0x5104, the field carries bit 15), 3 + D0 (0x6104),
// dC - 3 and dD - B (0x7324, negative; dD's field carries bit 15 when B = 6). z first:
// c = fma(fz, dC - 3, 1 + C0), d = fma(fz, dD - B, 3 + D0), x = fma(fx, d, c) is the edge value plus
// the bias b0 + fx k (b0 = 1 - 3 fz, k = 3 - B fz), the same for both edges: fx k is removed in the
// y-lerp, b0 once per atom by the caller (cell_lerp_b) or here (cell_lerp). The dummy cell (all
// fields zero) decodes to the bias itself: ~0 after the removal (within the rounding bound).
constexpr uint32_t kDecK = 0xC0403F00u;
__device__ __forceinline__ float dec_c0(uint32_t w) { return __uint_as_float(__byte_perm(w, kDecK, 0x5104)); }
__device__ __forceinline__ float dec_d0(uint32_t w) { return __uint_as_float(__byte_perm(w, kDecK, 0x6104)); }
__device__ __forceinline__ float dec_dz(uint32_t w) { return __uint_as_float(__byte_perm(w, kDecK, 0x7324)); }

struct CellBias {
  float k, b0;
};
__device__ __forceinline__ CellBias cell_bias(float fz, float nb) { return {fmaf(fz, nb, 3.0f), fmaf(fz, -3.0f, 1.0f)}; }

// quantised trilinear value + b0 (k from cell_bias of the same fz)
__device__ __forceinline__ float cell_lerp_b(const uint4 w, float fx, float fy, float fz, float k) {
  const float c0 = fmaf(fz, dec_dz(w.x), dec_c0(w.x));
  const float d0 = fmaf(fz, dec_dz(w.y), dec_d0(w.y));
  const float c1 = fmaf(fz, dec_dz(w.z), dec_c0(w.z));
  const float d1 = fmaf(fz, dec_dz(w.w), dec_d0(w.w));
  const float x0 = fmaf(fx, d0, c0), x1 = fmaf(fx, d1, c1);
  return fmaf(fy, x1 - x0, fmaf(fx, -k, x0));
}

__device__ __forceinline__ float cell_lerp(const uint4 w, float fx, float fy, float fz, float nb) {
  const CellBias cb = cell_bias(fz, nb);
  return cell_lerp_b(w, fx, fy, fz, cb.k) - cb.b0;
}

// One coarse sample at grid coordinates g: the quantised trilinear value when
// strictly inside the grid, else exactly 0 (the dummy cell). amin tracks the smallest L-inf
// distance of any sample to the grid boundary: a sample within the position bound of a face may be
// classified differently from the FP64 reference, so its candidate is re-scored exactly.
__device__ __forceinline__ float coarse_sample(const CoarseGrid& cg, float gx, float gy, float gz,
                                               float& amin) {
  const float e = fmaxf(fabsf(gx - cg.hx) - cg.hx, fmaxf(fabsf(gy - cg.hy) - cg.hy, fabsf(gz - cg.hz) - cg.hz));
  amin = fminf(amin, fabsf(e));
  const float rx = __fadd_rz(gx, kMagic), ry = __fadd_rz(gy, kMagic), rz = __fadd_rz(gz, kMagic);
  const float fx = gx - (rx - kMagic), fy = gy - (ry - kMagic), fz = gz - (rz - kMagic);
  const uint32_t cell = __float_as_uint(rx) + __float_as_uint(ry) * cg.cx + __float_as_uint(rz) * cg.cxy - cg.koff;
  return cell_lerp(cg.cells[e < 0.0f ? cell : cg.dummy], fx, fy, fz, cg.nb);
}

// coarse_sample that also tracks the smallest signed box distance (emin > ptol: clearly outside).
__device__ __forceinline__ float coarse_sample_e(const CoarseGrid& cg, float gx, float gy, float gz, float& amin,
                                                 float& emin) {
  const float e = fmaxf(fabsf(gx - cg.hx) - cg.hx, fmaxf(fabsf(gy - cg.hy) - cg.hy, fabsf(gz - cg.hz) - cg.hz));
  emin = fminf(emin, e);
  return coarse_sample(cg, gx, gy, gz, amin);
}

// coarse_sample for the separable alignment: the z coordinate's box term ez, fraction fz and cell
// plane offset zoff (already carrying -koff) are shared by the alpha rotations of a frame.
__device__ __forceinline__ float coarse_sample_z(const CoarseGrid& cg, float gx, float gy, float ez, float fz,
                                                 uint32_t zoff, float& amin) {
  const float e = fmaxf(fmaxf(fabsf(gx - cg.hx) - cg.hx, fabsf(gy - cg.hy) - cg.hy), ez);
  amin = fminf(amin, fabsf(e));
  const float rx = __fadd_rz(gx, kMagic), ry = __fadd_rz(gy, kMagic);
  const float fx = gx - (rx - kMagic), fy = gy - (ry - kMagic);
  const uint32_t cell = __float_as_uint(rx) + __float_as_uint(ry) * cg.cx + zoff;
  return cell_lerp(cg.cells[e < 0.0f ? cell : cg.dummy], fx, fy, fz, cg.nb);
}

// Interval form of coarse_sample for rotations with a sample near a face: a sample within ptol of
// the boundary may be inside or outside in FP64, so it contributes [0, v_in] with v_in sampled at
// the point clamped onto the grid (the clamp moves it by <= ptol, covered by one more eps).
__device__ __forceinline__ void coarse_sample_iv(const CoarseGrid& cg, float gx, float gy, float gz, float ptol,
                                                 float& lo, float& hi) {
  const float e = fmaxf(fabsf(gx - cg.hx) - cg.hx, fmaxf(fabsf(gy - cg.hy) - cg.hy, fabsf(gz - cg.hz) - cg.hz));
  if (e > ptol) return;
  float am = 0.f;
  const float v = coarse_sample(cg, fminf(fmaxf(gx, 0.f), 2.f * cg.hx - 1e-3f),
                                fminf(fmaxf(gy, 0.f), 2.f * cg.hy - 1e-3f),
                                fminf(fmaxf(gz, 0.f), 2.f * cg.hz - 1e-3f), am);
  hi += v;
  if (e < -ptol) lo += v;
}

// ------------------------------------------------------------------ K1b's FP32 field (GD_K1B_FIELDF)
// The coarse samples of the sweep straight from an FP32 copy of the field (8 corners, 7 lerps): no
// quantisation beyond the FP32 rounding of the values (q_eps_f), staged in shared memory when it
// fits (55 KB for 24^3) so the candidates' samples do not wait on L2 (the quantised cells, 195 KB,
// do not fit beside the warps' slots). A sample outside the grid reads the zero tail at `dummy`.
struct CoarseGridF {
  const float* f;       // shared (SC: a shared-window address in `base`) or global
  uint32_t base;        // SC: shared address of f
  float hx, hy, hz;     // half extents (dims-1)/2
  uint32_t nx, nxy;     // nodes per row / per plane
  uint32_t koff;        // 0x4B000000 * (1 + nx + nxy)
  uint32_t dummy;       // first float of the zero tail
};

template <bool SC>
__device__ __forceinline__ float load_f(const CoarseGridF& cg, uint32_t i) {
  if (SC) {
    float v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(cg.base + 4u * i));
    return v;
  }
  return __ldg(cg.f + i);
}

template <bool SC>
__device__ __forceinline__ float sample_f(const CoarseGridF& cg, float gx, float gy, float gz, float& amin,
                                          float& emin) {
  const float e = fmaxf(fabsf(gx - cg.hx) - cg.hx, fmaxf(fabsf(gy - cg.hy) - cg.hy, fabsf(gz - cg.hz) - cg.hz));
  emin = fminf(emin, e);
  amin = fminf(amin, fabsf(e));
  const float rx = __fadd_rz(gx, kMagic), ry = __fadd_rz(gy, kMagic), rz = __fadd_rz(gz, kMagic);
  const float fx = gx - (rx - kMagic), fy = gy - (ry - kMagic), fz = gz - (rz - kMagic);
  const uint32_t idx = __float_as_uint(rx) + __float_as_uint(ry) * cg.nx + __float_as_uint(rz) * cg.nxy - cg.koff;
  const uint32_t i = e < 0.0f ? idx : cg.dummy;
  const float c000 = load_f<SC>(cg, i), c100 = load_f<SC>(cg, i + 1), c010 = load_f<SC>(cg, i + cg.nx),
              c110 = load_f<SC>(cg, i + cg.nx + 1);
  const uint32_t j = i + cg.nxy;
  const float c001 = load_f<SC>(cg, j), c101 = load_f<SC>(cg, j + 1), c011 = load_f<SC>(cg, j + cg.nx),
              c111 = load_f<SC>(cg, j + cg.nx + 1);
  const float x00 = fmaf(fx, c100 - c000, c000), x10 = fmaf(fx, c110 - c010, c010);
  const float x01 = fmaf(fx, c101 - c001, c001), x11 = fmaf(fx, c111 - c011, c011);
  const float y0 = fmaf(fy, x10 - x00, x00), y1 = fmaf(fy, x11 - x01, x01);
  return fmaf(fz, y1 - y0, y0);
}

// ------------------------------------------------------------------ TMA staging
// Copy `bytes` from global to this CTA's shared memory with TMA bulk copies (cp.async.bulk,
// completion counted on an mbarrier): thread 0 arms the barrier with the byte count and issues the
// copies, every thread waits on the barrier's phase. Used for the once-per-CTA staging of the
// pocket cells and the FP64 field. Addresses or sizes that are not 16-byte multiples (an odd-size
// field) take a cooperative copy instead. Ends with a CTA barrier (the next call re-arms it).
__device__ __forceinline__ void stage_to_smem(void* dst, const void* src, uint32_t bytes) {
  __shared__ alignas(8) unsigned long long stage_bar;
  const uint32_t d = uint32_t(__cvta_generic_to_shared(dst));
  const uint32_t bar = uint32_t(__cvta_generic_to_shared(&stage_bar));
  const bool tma = bytes > 0 && bytes < (1u << 20) && ((d | uint32_t(reinterpret_cast<uintptr_t>(src)) | bytes) & 15u) == 0;
  if (tma) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      for (uint32_t off = 0; off < bytes; off += 65536u) {
        const uint32_t n = min(65536u, bytes - off);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(d + off), "l"(reinterpret_cast<const char*>(src) + off), "r"(n), "r"(bar)
                     : "memory");
      }
    }
    __syncthreads();  // the barrier is initialised before anyone polls it
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}"
        ::"r"(bar) : "memory");
    __syncthreads();  // every thread has seen the phase complete before the barrier is re-armed
    if (threadIdx.x == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
  } else {
    const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
    for (uint32_t i = threadIdx.x; i < bytes / 4u; i += blockDim.x) d32[i] = __ldg(s32 + i);
  }
  __syncthreads();
}

// ------------------------------------------------------------------ FP64 register pose helpers
template <int NS>
struct Pose {
  double x[NS], y[NS], z[NS];
};

template <int NS>
__device__ __forceinline__ V3d own(const Pose<NS>& P, int s) {
  return V3d{P.x[s], P.y[s], P.z[s]};
}

template <int NS>
__device__ __forceinline__ void set_own(Pose<NS>& P, int s, V3d v) {
  P.x[s] = v.x;
  P.y[s] = v.y;
  P.z[s] = v.z;
}

// Position of atom a (warp-uniform a) from its owner lane.
template <int NS>
__device__ __forceinline__ V3d fetch(const Pose<NS>& P, uint32_t a) {
  const int slot = int(a >> 5), src = int(a & 31);
  double vx = P.x[0], vy = P.y[0], vz = P.z[0];
#pragma unroll
  for (int s = 1; s < NS; ++s)
    if (slot == s) {
      vx = P.x[s];
      vy = P.y[s];
      vz = P.z[s];
    }
  return V3d{__shfl_sync(FULL, vx, src), __shfl_sync(FULL, vy, src), __shfl_sync(FULL, vz, src)};
}

// Index-order sums (the reference's left-to-right accumulation) through a per-warp shared
// scratch, so every lane gets the same bits: lanes deposit their values, lane c
// adds column c sequentially (LDS pipelined ahead of the dependent DADD chain), one shuffle
// broadcasts. A shuffle per term costs ~30 cycles of latency on the chain; an LDS does not.
__device__ __forceinline__ double serial_sum(const double* v, uint32_t n) {
  double sum = 0.0;
  uint32_t a = 0;
  for (; a + 4 <= n; a += 4) {
    const double v0 = v[a], v1 = v[a + 1], v2 = v[a + 2], v3 = v[a + 3];
    sum = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(sum, v0), v1), v2), v3);
  }
  for (; a < n; ++a) sum = __dadd_rn(sum, v[a]);
  return sum;
}

template <int NS>
__device__ __forceinline__ double ordered_sum_smem(const double (&v)[NS], uint32_t n, double* scr, uint32_t lane) {
#pragma unroll
  for (int s = 0; s < NS; ++s)
    if (lane + 32 * s < n) scr[lane + 32 * s] = v[s];
  __syncwarp();
  double sum = 0.0;
  if (lane == 0) sum = serial_sum(scr, n);
  sum = __shfl_sync(FULL, sum, 0);
  __syncwarp();
  return sum;
}

// centroid (geometry.cpp:40-46): index-order sums of x, y, z (lanes 0, 1, 2 in parallel) * (1/n).
// scr holds 3 n doubles.
template <int NS>
__device__ __forceinline__ V3d centroid_smem(const Pose<NS>& P, uint32_t n, double* scr, uint32_t lane) {
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const uint32_t a = lane + 32 * s;
    if (a < n) {
      scr[a] = P.x[s];
      scr[n + a] = P.y[s];
      scr[2 * n + a] = P.z[s];
    }
  }
  __syncwarp();
  double sum = 0.0;
  if (lane < 3) sum = serial_sum(scr + lane * n, n);
  const V3d tot{__shfl_sync(FULL, sum, 0), __shfl_sync(FULL, sum, 1), __shfl_sync(FULL, sum, 2)};
  __syncwarp();
  return vscale(__ddiv_rn(1.0, double(n)), tot);
}

// Element i of a small register array without a dynamic index (a dynamic index would put the
// array in local memory): a select chain over the NS slots.
template <int NS, class T>
__device__ __forceinline__ T pick(const T (&v)[NS], int i) {
  T r = v[0];
#pragma unroll
  for (int k = 1; k < NS; ++k)
    if (i == k) r = v[k];
  return r;
}
template <int NS, class T>
__device__ __forceinline__ void put(T (&v)[NS], int i, T x) {
#pragma unroll
  for (int k = 0; k < NS; ++k)
    if (i == k) v[k] = x;
}
template <int NS>
__device__ __forceinline__ void put2(uint32_t (&v)[NS][NS], int i, int j, uint32_t x) {
#pragma unroll
  for (int k = 0; k < NS; ++k)
#pragma unroll
    for (int l = 0; l < NS; ++l)
      if (i == k && j == l) v[k][l] = x;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

// Word w of a register bit set without dynamic indexing (a dynamic index would put the whole
// array in local memory).
template <int NW>
__device__ __forceinline__ uint32_t word_of(const uint32_t (&m)[NW], uint32_t w) {
  uint32_t v = m[0];
#pragma unroll
  for (int i = 1; i < NW; ++i)
    if (w == uint32_t(i)) v = m[i];
  return v;
}

template <int NW>
__device__ __forceinline__ bool bit4(const uint32_t (&m)[NW], uint32_t a) { return (word_of<NW>(m, a >> 5) >> (a & 31)) & 1u; }

// Bits [lo, hi) of a bit set, restricted to word w.
__device__ __forceinline__ uint32_t range_word(uint32_t w, uint32_t lo, uint32_t hi) {
  const int a = max(int(lo) - 32 * int(w), 0), e = min(int(hi) - 32 * int(w), 32);
  if (e <= a) return 0u;
  return (e >= 32 ? FULL : ((1u << e) - 1u)) & ~((1u << a) - 1u);
}

__device__ __forceinline__ Qd frag_quat(const double4& dt, V3d axis) {  // about_axis, geometry.hpp:46-50
  return Qd{dt.x, __dmul_rn(axis.x, dt.y), __dmul_rn(axis.y, dt.y), __dmul_rn(axis.z, dt.y)};
}

struct Item {
  uint32_t n, W, lig, rs;
  LigMeta m;
};

// The exact FP64 sampler and whole-rotation scorer are out-of-line: they run on rare paths and
// inlining them at every call site blew the kernel past the instruction cache.
#ifndef GD_SAMPLE_NOINLINE
#define GD_SAMPLE_NOINLINE 1
#endif
#if GD_SAMPLE_NOINLINE
__device__ __noinline__ double sample_exact_ni(const DevPocket& pk, V3d p) { return sample_exact(pk, p); }
#else
__device__ __forceinline__ double sample_exact_ni(const DevPocket& pk, V3d p) { return sample_exact(pk, p); }
#endif

// best_rotation_in_range's score of rotation q (docking.cpp:77-83), atoms in index order.
__device__ __noinline__ double exact_rotation_score(const DevPocket& pk, const double* gpose, uint32_t n, V3d cen,
                                                    Qd q) {
  double sum = 0.0;
  for (uint32_t a = 0; a < n; ++a) {
    const V3d p{gpose[3 * a], gpose[3 * a + 1], gpose[3 * a + 2]};
    sum = __dadd_rn(sum, sample_exact(pk, rotated_about(p, cen, q)));
  }
  return __ddiv_rn(sum, double(n));
}

#define GD_MO4(mo) (mo)[0], NS > 1 ? (mo)[NS > 1 ? 1 : 0] : 0u, NS > 2 ? (mo)[NS > 2 ? 2 : 0] : 0u, \
                   NS > 3 ? (mo)[NS > 3 ? 3 : 0] : 0u

// The exact paths of the dihedral sweep read the warp's FP64 pose X (3n doubles, atom order) and
// exact per-atom samples ES from its shared-memory slot: during the sweep the pose lives there,
// not in registers (register pressure of the step loop).

// Exact FP64 test of the non-bonded pairs of candidate k (rotate: M' atoms rotated by q about pi).
// cross_only: only pairs with exactly one atom in M' (the invariant pairs are known exactly).
#ifndef GD_EXACT_NOINLINE
#define GD_EXACT_NOINLINE 0
#endif
#if GD_EXACT_NOINLINE
#define GD_EXACT_FN __noinline__
#else
#define GD_EXACT_FN __forceinline__
#endif
template <int NS>
__device__ GD_EXACT_FN bool exact_clash_g(const DevBatch& b, uint32_t atom_base, uint32_t adj_base, uint32_t n,
                                           const double* X, uint32_t mo0, uint32_t mo1, uint32_t mo2, uint32_t mo3,
                                           bool rotate, V3d pi, Qd q, double clash, bool cross_only, uint32_t lane) {
  const uint32_t mo[4] = {mo0, mo1, mo2, mo3};
  const uint32_t W = (n + 31) >> 5;
  V3d pa[NS];
  double ra[NS];
#pragma unroll
  for (int t = 0; t < NS; ++t) {
    const uint32_t a = lane + 32 * t;
    pa[t] = V3d{0.0, 0.0, 0.0};
    ra[t] = 0.0;
    if (a < n) {
      pa[t] = V3d{X[3 * a], X[3 * a + 1], X[3 * a + 2]};
      ra[t] = b.atoms[atom_base + a].w;
      if (rotate && bit4<4>(mo, a)) pa[t] = rotated_about(pa[t], pi, q);
    }
  }
  bool hit = false;
  for (uint32_t bb = 0; bb < n; ++bb) {
    V3d pb{X[3 * bb], X[3 * bb + 1], X[3 * bb + 2]};
    const bool bm = bit4<4>(mo, bb);
    if (rotate && bm) pb = rotated_about(pb, pi, q);
    const double rb = b.atoms[atom_base + bb].w;
    const uint32_t* row = b.adj + adj_base + bb * W;
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const uint32_t a = lane + 32 * t;
      if (a >= n || a <= bb) continue;
      if (cross_only && bit4<4>(mo, a) == bm) continue;
      if ((__ldg(row + (a >> 5)) >> (a & 31)) & 1u) continue;
      hit |= pair_clash_exact(pa[t], pb, ra[t], rb, clash);
    }
  }
  return __any_sync(FULL, hit);
}

// Exact score of dihedral candidate k (score_pose, scoring.cpp:40-45): M' atoms rotated by q about
// pi and sampled in FP64 (none when rotate is false: the current pose, k = 0), the others from the
// exact per-atom cache, summed in atom order.
// scr[a] keeps every atom's value until the next call: the caller copies the moved atoms' new
// exact samples of its best candidate from there (a k != 0 commit stores them as the pose's ES).
template <int NS>
__device__ GD_EXACT_FN double exact_candidate_score_g(const DevPocket& pk, uint32_t n, const double* X,
                                                       const double* ES, uint32_t mo0, uint32_t mo1, uint32_t mo2,
                                                       uint32_t mo3, bool rotate, V3d pi, Qd q, uint32_t lane,
                                                       double* scr) {
  // lanes deposit their atoms' values straight into the index-order scratch (one copy of the
  // rotate + sample code: the slot loop is not unrolled, instruction-cache footprint)
#pragma unroll 1
  for (int t = 0; t < NS; ++t) {
    const uint32_t a = lane + 32 * t;
    const uint32_t mw = t == 0 ? mo0 : t == 1 ? mo1 : t == 2 ? mo2 : mo3;  // no dynamic array index
    if (a < n) {
      double v = ES[a];
      if (rotate && ((mw >> lane) & 1u))
        v = NS >= 4 ? sample_exact(pk, rotated_about(V3d{X[3 * a], X[3 * a + 1], X[3 * a + 2]}, pi, q))  // inline: C4 -7 %
                    : sample_exact_ni(pk, rotated_about(V3d{X[3 * a], X[3 * a + 1], X[3 * a + 2]}, pi, q));
      scr[a] = v;
    }
  }
  __syncwarp();
  double sum = 0.0;
  if (lane == 0) sum = serial_sum(scr, n);
  sum = __shfl_sync(FULL, sum, 0);
  __syncwarp();
  return __ddiv_rn(sum, double(n));
}

}  // namespace

// ============================================================================ K1a: coarse alignment
// Lean, high-occupancy kernel (no FP64 pose, no sweep state): per (ligand, restart) the FP32 start
// pose relative to its centroid, the coarse score and error bound of every grid rotation, and the
// list of rotations that can be the exact argmax (key_hi >= max key_lo - 2 eps),
// handed to K1b for the FP64 re-scoring. The start pose is built in FP32 here: its error (~1e-6 A
// for the rotation of p - c0, the centroid shift cancels in the relative coordinates) is far
// inside ptol, and only the coarse screen sees it.
template <int NS, int NT, bool SC>
__global__ void __launch_bounds__(NT, 1)
    align_coarse_kernel(DevPocket pk, DevParams pr, DevBatch b, uint32_t slot_floats) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t n_cells = pk.cell_dims[0] * pk.cell_dims[1] * pk.cell_dims[2];
  uint4* sc = reinterpret_cast<uint4*>(smem_raw);
  const uint4* cells = SC ? sc : pk.cells;
  float* slots = SC ? reinterpret_cast<float*>(sc + n_cells + 1) : reinterpret_cast<float*>(smem_raw);
  if (SC) {
#if GD_K1A_TMA_STAGE
    stage_to_smem(sc, pk.cells, (n_cells + 1) * uint32_t(sizeof(uint4)));
#else
    for (uint32_t i = threadIdx.x; i <= n_cells; i += blockDim.x) sc[i] = __ldg(pk.cells + i);
    __syncthreads();
#endif
  }
  float4* A = reinterpret_cast<float4*>(slots + size_t(warp) * slot_floats);
  const CoarseGrid cg{cells,
                      0.5f * float(pk.cell_dims[0]),
                      0.5f * float(pk.cell_dims[1]),
                      0.5f * float(pk.cell_dims[2]),
                      pk.cell_dims[0],
                      pk.cell_dims[0] * pk.cell_dims[1],
                      0x4B000000u * (1u + pk.cell_dims[0] + pk.cell_dims[0] * pk.cell_dims[1]),
                      n_cells,
                      -pk.dz_bias};
  const uint32_t N = pr.n_restarts;
  const uint64_t total = uint64_t(b.n_lig) * N;
  for (;;) {
    uint32_t item = 0;
    if (lane == 0) item = atomicAdd(b.work_counter + 1, 1u);
    item = __shfl_sync(FULL, item, 0);
    if (item >= total) break;
    if (b.order) item = b.order[item];  // claims in start-target order (launch_dock)
    const uint32_t lig = item / N;
    const LigMeta meta = b.meta[lig];
    const uint32_t n = meta.n;
    if (n > 32u * NS || n <= b.fast_min_n) continue;  // another launch's ligand (mixed batch)
    // start pose (docking.cpp:52-69): R(q) (p - c0) + t; only the part relative to its centroid
    // matters here, plus the centroid itself (t + mean of the rotated offsets, in FP64)
    float px[NS], py[NS], pz[NS];
    float sx = 0.f, sy = 0.f, sz = 0.f;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const uint32_t a = lane + 32 * s;
      px[s] = py[s] = pz[s] = 0.f;
      if (a < n) {
        const double4 at = b.atoms[meta.atom_base + a];
        px[s] = float(at.x);
        py[s] = float(at.y);
        pz[s] = float(at.z);
      }
      sx += px[s];
      sy += py[s];
      sz += pz[s];
    }
    const float inv_n = 1.0f / float(n);
    const float c0x = warp_sum(sx) * inv_n, c0y = warp_sum(sy) * inv_n, c0z = warp_sum(sz) * inv_n;
    const double4 q4 = b.start[2 * size_t(item)];
    const double4 t4 = b.start[2 * size_t(item) + 1];
    const float qw = float(q4.x), qx = float(q4.y), qy = float(q4.z), qz = float(q4.w);
    const float xx = qx * qx, yy = qy * qy, zz = qz * qz, xy = qx * qy, xz = qx * qz, yz = qy * qz;
    const float wx = qw * qx, wy = qw * qy, wz = qw * qz;
    const float m00 = 1.f - 2.f * (yy + zz), m01 = 2.f * (xy - wz), m02 = 2.f * (xz + wy);
    const float m10 = 2.f * (xy + wz), m11 = 1.f - 2.f * (xx + zz), m12 = 2.f * (yz - wx);
    const float m20 = 2.f * (xz - wy), m21 = 2.f * (yz + wx), m22 = 1.f - 2.f * (xx + yy);
    sx = sy = sz = 0.f;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const float vx = px[s] - c0x, vy = py[s] - c0y, vz = pz[s] - c0z;
      px[s] = fmaf(m00, vx, fmaf(m01, vy, m02 * vz));
      py[s] = fmaf(m10, vx, fmaf(m11, vy, m12 * vz));
      pz[s] = fmaf(m20, vx, fmaf(m21, vy, m22 * vz));
      if (lane + 32 * s < n) {
        sx += px[s];
        sy += py[s];
        sz += pz[s];
      }
    }
    const float cmx = warp_sum(sx) * inv_n, cmy = warp_sum(sy) * inv_n, cmz = warp_sum(sz) * inv_n;
    const V3d cen{t4.x + double(cmx), t4.y + double(cmy), t4.z + double(cmz)};
    const float tx = float(__ddiv_rn(__dsub_rn(cen.x, pk.origin[0]), pk.spacing));
    const float ty = float(__ddiv_rn(__dsub_rn(cen.y, pk.origin[1]), pk.spacing));
    const float tz = float(__ddiv_rn(__dsub_rn(cen.z, pk.origin[2]), pk.spacing));
    // Relative coordinates into A, "safe" atoms first: an atom at distance r from the centroid
    // stays within r of it under every rotation, so if that ball (plus 2e-3 grid units, far above
    // the FP32 error and ptol) is strictly inside the grid, every sample of it is inside and away
    // from the faces: its coarse samples need no box test. Order within A does
    // not matter for the coarse score (its error bound is order-free).
    // Class 0 (safe): the ball is inside in x, y and z. Class 1 (xy-safe): inside in x and y only,
    // so a sample's box term is its frame's z term (per atom, not per sample). Class 2: the rest.
    float ext = 0.f, vxs[NS], vys[NS], vzs[NS];
    uint32_t cls[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const uint32_t a = lane + 32 * s;
      vxs[s] = px[s] - cmx;
      vys[s] = py[s] - cmy;
      vzs[s] = pz[s] - cmz;
      const float r = sqrtf(fmaf(vxs[s], vxs[s], fmaf(vys[s], vys[s], vzs[s] * vzs[s])));
      const float rg = fmaf(r, pk.inv_spacing_f * (1.0f + 1e-5f), 2e-3f);
      const bool xy = tx - rg > 0.f && ty - rg > 0.f && tx + rg < 2.f * cg.hx && ty + rg < 2.f * cg.hy;
      const bool z = tz - rg > 0.f && tz + rg < 2.f * cg.hz;
      cls[s] = a >= n ? 3u : (xy ? (z ? 0u : 1u) : 2u);
      if (a < n) ext = fmaxf(ext, r);
    }
    uint32_t nsafe = 0, nxy = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      nsafe += __popc(__ballot_sync(FULL, cls[s] == 0u));
      nxy += __popc(__ballot_sync(FULL, cls[s] == 1u));
    }
    {
      uint32_t before[3] = {0u, nsafe, nsafe + nxy};
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const uint32_t a = lane + 32 * s;
        const uint32_t lt = (1u << lane) - 1u;
        uint32_t at = 0u;
#pragma unroll
        for (uint32_t c = 0; c < 3u; ++c) {
          const uint32_t bc = __ballot_sync(FULL, cls[s] == c);
          if (cls[s] == c) at = before[c] + __popc(bc & lt);
          before[c] += __popc(bc);
        }
        if (a < n) {
          A[at] = make_float4(vxs[s], vys[s], vzs[s], 0.f);
        } else if (a < meta.npad) {
          A[a] = make_float4(1e6f, 1e6f, 1e6f, 0.f);  // padding: far outside, contributes exactly 0
        }
      }
    }
    __syncwarp();
    // Position error bound (grid units, per axis) of every FP32 coordinate of this restart, as in
    // K1b; the ligand extent gets a 1e-3 grid-unit allowance for FP32 rounding.
    const float ext_g = warp_max(ext) * pk.inv_spacing_f + 1e-3f;
    const float maxdim = float(max(pk.dims[0], max(pk.dims[1], pk.dims[2])));
    const float ptol = 1.5e-5f + 5e-7f * maxdim + 6e-6f * ext_g;
    const float eps_s = pk.q_eps + 3.0f * pk.max_step * ptol;  // coarse per-sample error bound
    // coarse score error bound: per-sample FP32 rounding of the decode and lerps (<= 3e-6, values
    // below 8 in magnitude), the accumulation of n values carrying their bias b0 in [-2, 1] and of
    // the b0 themselves (partial sums below 2.1 n: <= 2.5e-7 n after the 1/n), the final scaling
    const float eps = eps_s + 3e-6f + 3e-7f * float(n) + 2e-7f;
    const float inv_n_scale = pk.coarse_scale / float(n);

    // ------------------------------------------------ coarse alignment sweep (all G rotations)
    // Lane l scores rotations g = l + 32 j. Per rotation the exact FP64 score lies in
    // [key_lo - eps, key_hi + eps] (key = coarse score, or for a rotation with a sample within ptol
    // of a face, the interval bounds from the second pass). Kept per lane: the KTOP largest key_hi,
    // the largest key_hi that was dropped, the largest key_lo. A rotation can be the exact argmax
    // only if key_hi >= max(key_lo) - 2 eps.
    float top_s[KTOP];
    uint32_t top_g[KTOP];
#pragma unroll
    for (int t = 0; t < KTOP; ++t) {
      top_s[t] = -1e30f;
      top_g[t] = 0xffffffffu;
    }
    float dropped = -1e30f, lkey = -1e30f;
    unsigned long long amb_mask = 0ull;  // rotations j (g = lane + 32 j) with a face-ambiguous sample
    const uint32_t npad = meta.npad;
    const bool big_grid = pr.G > 64u * 32u;
    // Separable form (default grids): R_g = Rz(alpha_i) F_f with frame f = j*c + k, g = i*b*c + f.
    // Lane l owns frames f = l + 32 m and all alpha of each; the frame's z row, its box term, floor
    // and cell plane are shared by the alpha rotations and x, y need a 2D rotation only.
    const uint32_t n_frames = pr.steps[1] * pr.steps[2];
    const bool separable = pr.steps[0] >= 8 && pr.steps[0] <= 16 && n_frames <= 128;
    // quarter-turn units (see the loop below): (kept frame, c0) in upload_grid_f's order
    const bool qt = separable && pr.steps[0] % (4 * kQtGroups) == 0;
    const uint32_t nq = pr.steps[0] / 4;
    static_assert(kQtGroups == 2 || kQtGroups == 4, "64-bit ambiguity masks: 4 kQtGroups bits per unit");
    const uint32_t n_units = qt ? pr.n_kept : 0u;
    const uint32_t n_full = n_units & ~31u, n_rem = n_units - n_full;
    const uint32_t gsz = n_rem <= 1u ? 32u : 32u >> (32 - __clz(n_rem - 1u));  // lanes per shared unit
    const uint32_t lgsz = 31u - __clz(gsz);
    const uint32_t n_iter = n_full / 32u + (n_rem ? 1u : 0u);
    const bool twins = qt && pr.n_twin_frames > 0;
    auto unit_of = [&](uint32_t mu) -> uint32_t { return mu * 32u >= n_full ? n_full + (lane >> lgsz) : lane + 32u * mu; };
    auto amb_to_g = [&](uint32_t bit) -> uint32_t {
      if (qt) {  // bit = 4 kQtGroups mu + 4 gi + q of the lane's unit mu
        const uint32_t u = unit_of(bit / (4u * kQtGroups));
        const uint32_t ue = __ldg(pr.frame_tab + n_frames + u);
        return ((ue >> 16) + ((bit >> 2) & (kQtGroups - 1u)) + (bit & 3u) * nq) * n_frames + (ue & 0xffffu);
      }
      return separable ? (bit & 15u) * n_frames + lane + 32u * (bit >> 4) : lane + 32u * bit;
    };
    // rotation g and its twins (rotations of the frames upload_grid_f folded into g's frame)
    auto twin_count = [&](uint32_t g) -> uint32_t {
      return twins ? (__ldg(pr.frame_tab + g % n_frames) & 0xffu) : 0u;
    };
    auto put_with_twins = [&](uint32_t at, uint32_t g) {
      uint16_t* cl = b.rs_cand + size_t(item) * kAlignCand;
      if (at < uint32_t(kAlignCand)) cl[at] = uint16_t(g);
      const uint32_t nt = twin_count(g);
      if (nt) {
        const uint32_t f0 = g % n_frames, ia = g / n_frames, e = __ldg(pr.frame_tab + f0) >> 8;
        for (uint32_t i = 0; i < nt; ++i) {
          const uint32_t tw = __ldg(pr.frame_tab + e + i);
          const uint32_t ia2 = (ia + pr.steps[0] - (tw >> 16)) % pr.steps[0];
          if (at + 1 + i < uint32_t(kAlignCand)) cl[at + 1 + i] = uint16_t(ia2 * n_frames + (tw & 0xffffu));
        }
      }
    };
    // collect mode (second pass): every rotation whose upper key reaches thr_c goes straight to
    // the restart's candidate list (rs_ncand counts them)
    bool collect = false;
    float thr_c = 0.f;
    auto insert = [&](float key_hi, uint32_t g) {
      if (collect) {
        if (key_hi >= thr_c) put_with_twins(uint32_t(atomicAdd(b.rs_ncand + item, int(1u + twin_count(g)))), g);
        return;
      }
      if (key_hi > top_s[KTOP - 1]) {
        dropped = fmaxf(dropped, top_s[KTOP - 1]);
        float vs = key_hi;
        uint32_t vg = g;
#pragma unroll
        for (int t = 0; t < KTOP; ++t) {  // sorted insert, descending
          if (vs > top_s[t]) {
            const float ts = top_s[t];
            const uint32_t tg = top_g[t];
            top_s[t] = vs;
            top_g[t] = vg;
            vs = ts;
            vg = tg;
          }
        }
      } else {
        dropped = fmaxf(dropped, key_hi);
      }
    };
    for (int pass = 0; pass < 2; ++pass) {
      if (qt) {
        // Quarter-turn symmetry: alpha_{c + q na/4} = alpha_c + q pi/2, so one 2D rotation
        // (rx, ry) = Rz(alpha_c) (wx, wy) gives the four samples t + (rx, ry), t + (-ry, rx),
        // t - (rx, ry), t + (ry, -rx): two FADDs per sample for x, y. kQtGroups consecutive c share
        // one pass over the atoms (the frame transform and the z terms are per atom).
        // byte offset of a cell from the three RZ-floor bit patterns: 16 bx + 16 cx by + zoff16
        const uint32_t cx16 = cg.cx * 16u, cxy16 = cg.cxy * 16u;
        // (shared: absolute 32-bit shared addresses; global: byte offsets from cg.cells)
        const uint32_t base16 = (SC ? uint32_t(__cvta_generic_to_shared(cg.cells)) : 0u) - cg.koff * 16u;
        const uint32_t dummy16 = (SC ? uint32_t(__cvta_generic_to_shared(cg.cells)) : 0u) + cg.dummy * 16u;
        // Work units: (kept frame, kQtGroups consecutive quarter-turn groups), 8 rotations each; twin
        // frames (the same rotations as a kept frame's, upload_grid_f) are not screened: their
        // rotations enter the candidate list with their twin's. Lane l takes units l + 32 mu; the
        // n_rem units beyond the last full round are shared by groups of gsz lanes (atoms split
        // over the group, partial sums combined by shuffles), so no lane screens a ninth unit
        // while others idle.
        for (uint32_t mu = 0; mu < n_iter; ++mu) {
          const bool coop = mu * 32u >= n_full;  // warp-uniform
          const uint32_t gs = coop ? gsz : 1u, sub = coop ? (lane & (gsz - 1u)) : 0u;
          const uint32_t u = coop ? n_full + (lane >> lgsz) : lane + 32u * mu;
          const bool active = u < n_units;
          const uint32_t ue = active ? __ldg(pr.frame_tab + n_frames + u) : 0u;
          const uint32_t f = ue & 0xffffu, c0 = ue >> 16;
          const float4 F0 = __ldg(pr.frames + 3 * f), F1 = __ldg(pr.frames + 3 * f + 1), F2 = __ldg(pr.frames + 3 * f + 2);
          {
            float acc[4 * kQtGroups], amn[4 * kQtGroups];
            float2 cs[kQtGroups];
  #pragma unroll
            for (int i = 0; i < 4 * kQtGroups; ++i) {
              acc[i] = 0.f;
              amn[i] = 1e30f;
            }
  #pragma unroll
            for (int gi = 0; gi < kQtGroups; ++gi) cs[gi] = pr.acs[(c0 + gi) & 15];
            // one atom of class CLS (see above): 0 skips the box test, the face tracking and the
            // dummy select; 1 uses its frame's z term for all its samples (one face-tracking update
            // per atom, a select per sample); 2 tests every sample
            float amz = 1e30f, bsum = 0.f;
            float2 acc2[2 * kQtGroups];
  #pragma unroll
            for (int i = 0; i < 2 * kQtGroups; ++i) acc2[i] = make_float2(0.f, 0.f);
            float2 cs_a[kQtGroups], cs_b[kQtGroups], cs_c[kQtGroups];  // (c, -s), (-s, -c), (s, c)
  #pragma unroll
            for (int gi = 0; gi < kQtGroups; ++gi) {
              cs_a[gi] = make_float2(cs[gi].x, -cs[gi].y);
              cs_b[gi] = make_float2(-cs[gi].y, -cs[gi].x);
              cs_c[gi] = make_float2(cs[gi].y, cs[gi].x);
            }
            const float2 T2x = make_float2(tx, tx), T2y = make_float2(ty, ty);
            const float2 M2 = make_float2(kMagic, kMagic), N12 = make_float2(-1.f, -1.f);
            auto atom2 = [&](uint32_t a, auto cls_tag) {
              constexpr int CLS = decltype(cls_tag)::value;
              const float4 v = A[a];
              const float wx = fmaf(F0.x, v.x, fmaf(F0.y, v.y, F0.z * v.z));
              const float wy = fmaf(F1.x, v.x, fmaf(F1.y, v.y, F1.z * v.z));
              const float gz = fmaf(F2.x, v.x, fmaf(F2.y, v.y, fmaf(F2.z, v.z, tz)));
              const float ez = CLS == 0 ? 0.f : fabsf(gz - cg.hz) - cg.hz;
              if (CLS == 1) amz = fminf(amz, fabsf(ez));
              const float rz = __fadd_rz(gz, kMagic);
              const float fz = gz - (rz - kMagic);
              const uint32_t zoff16 = __float_as_uint(rz) * cxy16 + base16;
              const CellBias cb = cell_bias(fz, cg.nb);
              bsum += cb.b0;
              const float2 FZ = make_float2(fz, fz), NK = make_float2(-cb.k, -cb.k);
              const float2 WX = make_float2(wx, wx), WY = make_float2(wy, wy);
  #pragma unroll
              for (int gi = 0; gi < kQtGroups; ++gi) {
                // (rx, -ry) and (ry, rx): rx = c wx - s wy, ry = s wx + c wy (as the scalar form)
                const float2 X01 = __ffma2_rn(WX, cs_a[gi], __fmul2_rn(WY, cs_b[gi]));
                const float2 Y01 = __ffma2_rn(WX, cs_c[gi], __fmul2_rn(WY, cs_a[gi]));
  #pragma unroll
                for (int h = 0; h < 2; ++h) {
                  // samples q = 2h, 2h + 1: t + (rx, ry), t + (-ry, rx) | t - (rx, ry), t + (ry, -rx)
                  // (differences as fma(a, -1, b): the same rounding as b - a, without separate negations)
                  const float2 gx = h == 0 ? __fadd2_rn(T2x, X01) : __ffma2_rn(X01, N12, T2x);
                  const float2 gy = h == 0 ? __fadd2_rn(T2y, Y01) : __ffma2_rn(Y01, N12, T2y);
                  const float2 rX = __fadd2_rz(gx, M2), rY = __fadd2_rz(gy, M2);
                  const float2 ntX = __ffma2_rn(rX, N12, M2), ntY = __ffma2_rn(rY, N12, M2);  // -floor(g), exact
                  const float2 fX = __fadd2_rn(gx, ntX);
                  const float2 fY = __fadd2_rn(gy, ntY);
                  uint32_t ad0 = __float_as_uint(rY.x) * cx16 + (__float_as_uint(rX.x) * 16u + zoff16);
                  uint32_t ad1 = __float_as_uint(rY.y) * cx16 + (__float_as_uint(rX.y) * 16u + zoff16);
                  if (CLS == 1) {
                    ad0 = ez < 0.0f ? ad0 : dummy16;
                    ad1 = ez < 0.0f ? ad1 : dummy16;
                  }
                  if (CLS == 2) {
                    const float e0 = fmaxf(fmaxf(fabsf(gx.x - cg.hx) - cg.hx, fabsf(gy.x - cg.hy) - cg.hy), ez);
                    const float e1 = fmaxf(fmaxf(fabsf(gx.y - cg.hx) - cg.hx, fabsf(gy.y - cg.hy) - cg.hy), ez);
                    amn[4 * gi + 2 * h] = fminf(amn[4 * gi + 2 * h], fabsf(e0));
                    amn[4 * gi + 2 * h + 1] = fminf(amn[4 * gi + 2 * h + 1], fabsf(e1));
                    ad0 = e0 < 0.0f ? ad0 : dummy16;
                    ad1 = e1 < 0.0f ? ad1 : dummy16;
                  }
                  const uint4 wA = load_cell<SC>(cg, ad0), wB = load_cell<SC>(cg, ad1);
                  const float2 c0 = __ffma2_rn(FZ, make_float2(dec_dz(wA.x), dec_dz(wB.x)), make_float2(dec_c0(wA.x), dec_c0(wB.x)));
                  const float2 d0 = __ffma2_rn(FZ, make_float2(dec_dz(wA.y), dec_dz(wB.y)), make_float2(dec_d0(wA.y), dec_d0(wB.y)));
                  const float2 c1 = __ffma2_rn(FZ, make_float2(dec_dz(wA.z), dec_dz(wB.z)), make_float2(dec_c0(wA.z), dec_c0(wB.z)));
                  const float2 d1 = __ffma2_rn(FZ, make_float2(dec_dz(wA.w), dec_dz(wB.w)), make_float2(dec_d0(wA.w), dec_d0(wB.w)));
                  const float2 x0 = __ffma2_rn(fX, d0, c0), x1 = __ffma2_rn(fX, d1, c1);
                  const float2 dx = __ffma2_rn(x0, N12, x1);
                  const float2 r = __ffma2_rn(fY, dx, __ffma2_rn(fX, NK, x0));
                  acc2[2 * gi + h] = __fadd2_rn(acc2[2 * gi + h], r);
                }
              }
            };
            if (active) {
              // the samples in pairs (quarter-turns q = 2h, 2h + 1 of one group) through the f32x2 pipe
  #pragma unroll 1
              for (uint32_t a = sub; a < nsafe; a += gs) atom2(a, std::integral_constant<int, 0>{});
  #pragma unroll 1
              for (uint32_t a = nsafe + ((sub - nsafe) & (gs - 1u)); a < nsafe + nxy; a += gs)
                atom2(a, std::integral_constant<int, 1>{});
  #pragma unroll 1
              for (uint32_t a = nsafe + nxy + ((sub - nsafe - nxy) & (gs - 1u)); a < n; a += gs)
                atom2(a, std::integral_constant<int, 2>{});
            }
            if (coop) {  // combine the group's partial sums (any order: the error bound is order-free)
              for (uint32_t o = 1; o < gsz; o <<= 1) {
  #pragma unroll
                for (int i = 0; i < 2 * kQtGroups; ++i) {
                  acc2[i].x += __shfl_xor_sync(FULL, acc2[i].x, o);
                  acc2[i].y += __shfl_xor_sync(FULL, acc2[i].y, o);
                }
  #pragma unroll
                for (int i = 0; i < 4 * kQtGroups; ++i) amn[i] = fminf(amn[i], __shfl_xor_sync(FULL, amn[i], o));
                bsum += __shfl_xor_sync(FULL, bsum, o);
                amz = fminf(amz, __shfl_xor_sync(FULL, amz, o));
              }
            }
  #pragma unroll
            for (int i = 0; i < 2 * kQtGroups; ++i) {
              acc[2 * i] = acc2[i].x;
              acc[2 * i + 1] = acc2[i].y;
            }
            if (active && sub == 0u) {
  #pragma unroll
              for (int i = 0; i < 4 * kQtGroups; ++i) amn[i] = fminf(amn[i], amz);
  #pragma unroll
              for (int gi = 0; gi < kQtGroups; ++gi)
  #pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const uint32_t ia = c0 + gi + q * nq;
                  const float sc = (acc[4 * gi + q] - bsum) * inv_n_scale;
                  if (amn[4 * gi + q] <= ptol) {
                    amb_mask |= 1ull << (4u * kQtGroups * mu + 4u * gi + q);
                  } else {
                    insert(sc, ia * n_frames + f);
                    lkey = fmaxf(lkey, sc);
                  }
                }
            }
          }
        }
      } else if (separable) {
        const uint32_t na = pr.steps[0];
        for (uint32_t f = lane, m = 0; f < n_frames; f += 32, ++m) {
          const float4 F0 = __ldg(pr.frames + 3 * f), F1 = __ldg(pr.frames + 3 * f + 1), F2 = __ldg(pr.frames + 3 * f + 2);
          // alpha in chunks of kAlphaChunk (the frame transform is redone per chunk) so the unrolled
          // body stays small enough for the instruction cache
  #pragma unroll 1
          for (uint32_t i0 = 0; i0 < na; i0 += kAlphaChunk) {
            float acc[kAlphaChunk], amn[kAlphaChunk];
            float2 cs[kAlphaChunk];
  #pragma unroll
            for (int i = 0; i < kAlphaChunk; ++i) {
              acc[i] = 0.f;
              amn[i] = 1e30f;
              cs[i] = pr.acs[(i0 + i) & 15];
            }
  #pragma unroll 1
            for (uint32_t a = 0; a < npad; ++a) {
              const float4 v = A[a];
              const float wx = fmaf(F0.x, v.x, fmaf(F0.y, v.y, F0.z * v.z));
              const float wy = fmaf(F1.x, v.x, fmaf(F1.y, v.y, F1.z * v.z));
              const float gz = fmaf(F2.x, v.x, fmaf(F2.y, v.y, fmaf(F2.z, v.z, tz)));
              const float ez = fabsf(gz - cg.hz) - cg.hz;
              const float rz = __fadd_rz(gz, kMagic);
              const float fz = gz - (rz - kMagic);
              const uint32_t zoff = __float_as_uint(rz) * cg.cxy - cg.koff;
  #pragma unroll
              for (int i = 0; i < kAlphaChunk; ++i) {
                const float gx = fmaf(cs[i].x, wx, fmaf(-cs[i].y, wy, tx));
                const float gy = fmaf(cs[i].y, wx, fmaf(cs[i].x, wy, ty));
                acc[i] += coarse_sample_z(cg, gx, gy, ez, fz, zoff, amn[i]);
              }
            }
  #pragma unroll
            for (int i = 0; i < kAlphaChunk; ++i) {
              const uint32_t ia = i0 + i;
              if (ia >= na) break;
              const float sc = acc[i] * inv_n_scale;
              if (amn[i] <= ptol) {
                amb_mask |= 1ull << (16 * m + ia);
              } else {
                insert(sc, ia * n_frames + f);
                lkey = fmaxf(lkey, sc);
              }
            }
          }
        }
      } else {
        for (uint32_t g = lane, j = 0; g < pr.G; g += 32, ++j) {
          const float4 r0 = __ldg(pr.grid_f + 3 * g), r1 = __ldg(pr.grid_f + 3 * g + 1), r2 = __ldg(pr.grid_f + 3 * g + 2);
          float acc0 = 0.f, acc1 = 0.f, amin = 1e30f;
  #pragma unroll kAlignUnroll
          for (uint32_t a = 0; a < npad; a += 4) {
            const float4 v0 = A[a], v1 = A[a + 1], v2 = A[a + 2], v3 = A[a + 3];
            acc0 += coarse_sample(cg, fmaf(r0.x, v0.x, fmaf(r0.y, v0.y, fmaf(r0.z, v0.z, tx))),
                                  fmaf(r1.x, v0.x, fmaf(r1.y, v0.y, fmaf(r1.z, v0.z, ty))),
                                  fmaf(r2.x, v0.x, fmaf(r2.y, v0.y, fmaf(r2.z, v0.z, tz))), amin);
            acc1 += coarse_sample(cg, fmaf(r0.x, v1.x, fmaf(r0.y, v1.y, fmaf(r0.z, v1.z, tx))),
                                  fmaf(r1.x, v1.x, fmaf(r1.y, v1.y, fmaf(r1.z, v1.z, ty))),
                                  fmaf(r2.x, v1.x, fmaf(r2.y, v1.y, fmaf(r2.z, v1.z, tz))), amin);
            acc0 += coarse_sample(cg, fmaf(r0.x, v2.x, fmaf(r0.y, v2.y, fmaf(r0.z, v2.z, tx))),
                                  fmaf(r1.x, v2.x, fmaf(r1.y, v2.y, fmaf(r1.z, v2.z, ty))),
                                  fmaf(r2.x, v2.x, fmaf(r2.y, v2.y, fmaf(r2.z, v2.z, tz))), amin);
            acc1 += coarse_sample(cg, fmaf(r0.x, v3.x, fmaf(r0.y, v3.y, fmaf(r0.z, v3.z, tx))),
                                  fmaf(r1.x, v3.x, fmaf(r1.y, v3.y, fmaf(r1.z, v3.z, ty))),
                                  fmaf(r2.x, v3.x, fmaf(r2.y, v3.y, fmaf(r2.z, v3.z, tz))), amin);
          }
          const float sc = (acc0 + acc1) * inv_n_scale;
          if (amin <= ptol) {
            amb_mask |= (j < 64 ? 1ull << j : 0ull);
            if (j >= 64) lkey = 1e30f;  // cannot track: forces the exact fallback below
          } else {
            insert(sc, g);
            lkey = fmaxf(lkey, sc);
          }
        }
      }
      // second pass over face-ambiguous rotations: interval bounds (rare; z-face ambiguities come
      // in groups of 16 rotations that share (beta, gamma) and therefore the z coordinate)
      for (unsigned long long mk = amb_mask; mk; mk &= mk - 1) {
        const uint32_t g = amb_to_g(uint32_t(__ffsll(static_cast<long long>(mk)) - 1));
        const float4 r0 = __ldg(pr.grid_f + 3 * g), r1 = __ldg(pr.grid_f + 3 * g + 1), r2 = __ldg(pr.grid_f + 3 * g + 2);
        float lo = 0.f, hi = 0.f;
  #pragma unroll 1
        for (uint32_t a = 0; a < npad; ++a) {
          const float4 v = A[a];
          coarse_sample_iv(cg, fmaf(r0.x, v.x, fmaf(r0.y, v.y, fmaf(r0.z, v.z, tx))),
                           fmaf(r1.x, v.x, fmaf(r1.y, v.y, fmaf(r1.z, v.z, ty))),
                           fmaf(r2.x, v.x, fmaf(r2.y, v.y, fmaf(r2.z, v.z, tz))), ptol, lo, hi);
        }
        insert(hi * inv_n_scale + eps, g);  // one extra eps for the clamp
        lkey = fmaxf(lkey, lo * inv_n_scale);
      }
      if (collect) {
        __syncwarp();
        if (lane == 0 && atomicAdd(b.rs_ncand + item, 0) > kAlignCand) b.rs_ncand[item] = -1;
        break;
      }
      const float B = warp_max(lkey);
      // a twin's exact score differs from its kept rotation's by FP64 rounding of the quaternions
      // (~1e-16): 1e-7 below the threshold covers it
      const float thr = B - 2.0f * eps - (twins ? 1e-7f : 0.f);
      const bool dropped_any = __any_sync(FULL, dropped >= thr);
      const bool hard = B < -1e29f || B > 1e29f || big_grid;
      // candidate list for K1b (order irrelevant: K1b takes max exact score, lowest index)
      uint32_t cnt = 0;
      if (!dropped_any && !hard) {
#pragma unroll
        for (int t = 0; t < KTOP; ++t) {
          const bool c = top_s[t] >= thr;
          const uint32_t k = c ? 1u + twin_count(top_g[t]) : 0u;  // entries: the rotation and its twins
          uint32_t incl = k;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= uint32_t(o)) incl += y;
          }
          if (c) put_with_twins(cnt + incl - k, top_g[t]);
          cnt += __shfl_sync(FULL, incl, 31);
        }
      }
      if (!dropped_any || hard) {
        if (lane == 0) b.rs_ncand[item] = (dropped_any || hard || cnt > uint32_t(kAlignCand)) ? -1 : int32_t(cnt);
        break;
      }
      // A lane kept only its KTOP best keys and dropped one that reaches thr (several near-equal
      // alphas of one frame): a second pass with the threshold known collects every candidate
      // (rare: ~1 restart in 8000 on C2; far cheaper than K1b's all-FP64 alignment).
      collect = true;
      thr_c = thr;
      if (lane == 0) {
        atomicExch(b.rs_ncand + item, 0);
        atomicAdd(b.stats + 6, 1ull);
      }
      __syncwarp();
      amb_mask = 0ull;
    }
  }
}


// ============================================================================ K1r: exact alignment
// Per (ligand, restart): the FP64 start pose (docking.cpp:52-69), K1a's candidate rotations
// re-scored in the reference's arithmetic (best_rotation_in_range + combine, docking.cpp:71-108;
// every rotation when K1a handed over the restart), apply_rotation_choice (docking.cpp:110-118),
// and the exact per-atom samples of the aligned pose: handed to K1b through HBM (rs_pose, rs_es),
// so the sweep kernel holds only the sweep (its instruction footprint). Warp per
// restart, pose in the warp's shared slot (3 n doubles) + 3 n doubles of index-order scratch.
template <int NS, int NT>
__global__ void __launch_bounds__(NT, 1)
    align_refine_kernel(DevPocket pk_in, DevParams pr, DevBatch b, uint32_t slot_doubles, uint32_t field_in_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ DevPocket spk;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) spk = pk_in;
  __syncthreads();
  DevPocket& pk = spk;
  double* slots = reinterpret_cast<double*>(smem_raw);
  if (field_in_smem) {
    double* sf = slots + size_t(blockDim.x >> 5) * slot_doubles;
    const uint32_t nv = pk.dims[0] * pk.dims[1] * pk.dims[2];
    stage_to_smem(sf, pk_in.field, nv * uint32_t(sizeof(double)));
    if (threadIdx.x == 0) pk.field = sf;
    __syncthreads();
  }
  const uint32_t npad = (b.max_n + 3) & ~3u;
  double* X = slots + size_t(warp) * slot_doubles;  // pose, atom order
  double* SCR = X + 3 * npad;                       // index-order sums
  const uint32_t N = pr.n_restarts;
  const uint64_t total = uint64_t(b.n_lig) * N;
  uint32_t st_aexact = 0, st_afall = 0;
  // centroid (geometry.cpp:40-46) of the pose in X: index-order sums of x, y, z (lanes 0, 1, 2)
  // times 1/n
  auto centroid = [&](uint32_t n) -> V3d {
    double sum = 0.0;
    if (lane < 3)
      for (uint32_t a = 0; a < n; ++a) sum = __dadd_rn(sum, X[3 * a + lane]);
    const V3d tot{__shfl_sync(FULL, sum, 0), __shfl_sync(FULL, sum, 1), __shfl_sync(FULL, sum, 2)};
    return vscale(__ddiv_rn(1.0, double(n)), tot);
  };
  for (;;) {
    uint32_t item = 0;
    if (lane == 0) item = atomicAdd(b.work_counter + 3, 1u);
    item = __shfl_sync(FULL, item, 0);
    if (item >= total) break;
    if (b.order) item = b.order[item];
    const uint32_t lig = item / N, rs = item - lig * N;
    const LigMeta m = b.meta[lig];
    const uint32_t n = m.n;
    if (n > 32u * NS || n <= b.fast_min_n) continue;  // another launch's ligand (mixed batch)
    // ---- starting pose (docking.cpp:52-69): r.apply(p - centroid) + target, FP64
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const uint32_t a = lane + 32 * s;
      if (a < n) {
        const double4 at = b.atoms[m.atom_base + a];
        X[3 * a] = at.x;
        X[3 * a + 1] = at.y;
        X[3 * a + 2] = at.z;
      }
    }
    __syncwarp();
    {
      const V3d c0 = centroid(n);
      const double4 q4 = b.start[2 * size_t(item)];
      const double4 t4 = b.start[2 * size_t(item) + 1];
      const Qd qs{q4.x, q4.y, q4.z, q4.w};
      const V3d tgt{t4.x, t4.y, t4.z};
      __syncwarp();
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const uint32_t a = lane + 32 * s;
        if (a < n) {
          const V3d v = vadd(qapply(qs, vsub(V3d{X[3 * a], X[3 * a + 1], X[3 * a + 2]}, c0)), tgt);
          X[3 * a] = v.x;
          X[3 * a + 1] = v.y;
          X[3 * a + 2] = v.z;
        }
      }
      __syncwarp();
    }
    const V3d cen = centroid(n);  // best_rotation_in_range's centroid (docking.cpp:76)
    // the ligand extent about the centroid: K1b's position error bound
    float ext = 0.f;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const uint32_t a = lane + 32 * s;
      if (a < n) {
        const V3d v = vsub(V3d{X[3 * a], X[3 * a + 1], X[3 * a + 2]}, cen);
        ext = fmaxf(ext, float(__dsqrt_rn(vdot(v, v))));
      }
    }
    ext = warp_max(ext);
    // ---- exact FP64 re-scoring of K1a's candidates, or (ncand < 0) of every rotation
    const int32_t ncand = b.rs_ncand[item];
    double best_s = -1.0;
    uint32_t best_g = 0xffffffffu;
    if (ncand < 0 || pr.G > 65535u) {
      ++st_afall;
      for (uint32_t g = lane; g < pr.G; g += 32) {
        const double4 gq = pr.grid[g];
        const double sc = exact_rotation_score(pk, X, n, cen, Qd{gq.x, gq.y, gq.z, gq.w});
        if (best_g == 0xffffffffu || sc > best_s) {  // g ascending within a lane: first max wins
          best_s = sc;
          best_g = g;
        }
      }
    } else {
      // warp-cooperative: candidates one at a time, lanes over atoms, index-order sum / n
      static_assert(kAlignCand <= 64, "two candidate words per lane");
      const uint16_t* cl = b.rs_cand + size_t(item) * kAlignCand;
      const uint32_t my_g0 = lane < uint32_t(ncand) ? cl[lane] : 0u;
      const uint32_t my_g1 = lane + 32 < uint32_t(ncand) ? cl[lane + 32] : 0u;
      for (int32_t c = 0; c < ncand; ++c) {
        const uint32_t g = __shfl_sync(FULL, c < 32 ? my_g0 : my_g1, c & 31);
        ++st_aexact;
        const double4 gq = pr.grid[g];
        const double sc = exact_candidate_score_g<NS>(pk, n, X, SCR, FULL, FULL, FULL, FULL, true, cen,
                                                      Qd{gq.x, gq.y, gq.z, gq.w}, lane, SCR);
        if (best_g == 0xffffffffu || sc > best_s || (sc == best_s && g < best_g)) {
          best_s = sc;
          best_g = g;
        }
      }
    }
    for (int off = 16; off > 0; off >>= 1) {  // combine (docking.cpp:93-108)
      const double os = __shfl_xor_sync(FULL, best_s, off);
      const uint32_t og = __shfl_xor_sync(FULL, best_g, off);
      if (og != 0xffffffffu && (best_g == 0xffffffffu || os > best_s || (os == best_s && og < best_g))) {
        best_s = os;
        best_g = og;
      }
    }
    // ---- apply_rotation_choice (docking.cpp:110-118) + the exact samples of the aligned pose
    {
      const double4 gq = pr.grid[best_g];
      const Qd q{gq.x, gq.y, gq.z, gq.w};
      const size_t base = size_t(m.atom_base) * N + size_t(rs) * n;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const uint32_t a = lane + 32 * s;
        if (a < n) {
          const V3d v = rotated_about(V3d{X[3 * a], X[3 * a + 1], X[3 * a + 2]}, cen, q);
          b.rs_pose[3 * (base + a)] = v.x;
          b.rs_pose[3 * (base + a) + 1] = v.y;
          b.rs_pose[3 * (base + a) + 2] = v.z;
          b.rs_es[base + a] = sample_exact_ni(pk, v);
        }
      }
    }
    if (lane == 0) {
      b.rs_align_index[item] = best_g;
      b.rs_align_score[item] = best_s;
      b.rs_ext[item] = ext;
    }
    __syncwarp();
  }
  if (lane == 0) {
    atomicAdd(b.stats + 1, (unsigned long long)st_aexact);
    atomicAdd(b.stats + 2, (unsigned long long)st_afall);
  }
}

// ============================================================================ the kernel
// NT = threads per CTA (launch bound): 64 registers at 1024 threads spilled the smem bases inside
// the hot loops, so the kernel trades warps for registers.
template <int NS, int NT, bool SC>
__global__ void __launch_bounds__(NT, 1)
    dock_fast_kernel(DevPocket pk_in, DevParams pr, DevBatch b, uint32_t slot_floats, uint32_t field_in_smem) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  // One DevPocket per CTA in shared memory (with the field pointer redirected below): the exact
  // samplers take it by reference, and a per-thread copy would live in local memory
  __shared__ DevPocket spk;
  __shared__ uint32_t sweep_ctr[32][kSweepCtr];  // per warp: executed sweep work, see st_* below
  if (threadIdx.x == 0) spk = pk_in;
  if (threadIdx.x < 32 * kSweepCtr) sweep_ctr[threadIdx.x / kSweepCtr][threadIdx.x % kSweepCtr] = 0u;
  __syncthreads();
  DevPocket& pk = spk;
  const uint32_t n_cells = pk.cell_dims[0] * pk.cell_dims[1] * pk.cell_dims[2];
  // SC: the pocket cells are staged once per CTA into shared memory (every warp of every work item
  // reads them; a compile-time flag so the gather is an LDS.128, not a generic load)
#if GD_K1B_FIELDF
  // SC: the FP32 field (+ zero tail) behind the warp slots, the coarse samples' source; else the
  // quantised cells through L1/L2. The FP64 field after it when it fits.
  const uint4* cells = pk.cells;
  float* slots = reinterpret_cast<float*>(smem_raw);
  float* sff = slots + size_t(blockDim.x >> 5) * slot_floats;
  if (SC) stage_to_smem(sff, pk.field_f, pk.f_count * uint32_t(sizeof(float)));
  const CoarseGridF cgf{SC ? sff : pk.field_f,
                        SC ? uint32_t(__cvta_generic_to_shared(sff)) : 0u,
                        0.5f * float(pk.cell_dims[0]),
                        0.5f * float(pk.cell_dims[1]),
                        0.5f * float(pk.cell_dims[2]),
                        pk.dims[0],
                        pk.dims[0] * pk.dims[1],
                        0x4B000000u * (1u + pk.dims[0] + pk.dims[0] * pk.dims[1]),
                        pk.f_dummy};
  if (field_in_smem) {
    double* sf = reinterpret_cast<double*>(sff + (SC ? ((pk.f_count + 3u) & ~3u) : 0u));
    const uint32_t nv = pk.dims[0] * pk.dims[1] * pk.dims[2];
#else
  uint4* sc = reinterpret_cast<uint4*>(smem_raw);
  const uint4* cells = SC ? sc : pk.cells;
  float* slots = SC ? reinterpret_cast<float*>(sc + n_cells + 1) : reinterpret_cast<float*>(smem_raw);
  if (SC) stage_to_smem(sc, pk.cells, (n_cells + 1) * uint32_t(sizeof(uint4)));
  if (field_in_smem) {
    // the FP64 field (exact samples of the refinement, refresh and exact decisions) behind the
    // warp slots: shared-memory latency instead of L2 for every exact sample
    double* sf = reinterpret_cast<double*>(slots + size_t(blockDim.x >> 5) * slot_floats);
    const uint32_t nv = pk.dims[0] * pk.dims[1] * pk.dims[2];
#endif
    stage_to_smem(sf, pk_in.field, nv * uint32_t(sizeof(double)));
    if (threadIdx.x == 0) pk.field = sf;
    __syncthreads();
  }
  float4* A = reinterpret_cast<float4*>(slots + size_t(warp) * slot_floats);
  // Behind the atom slot, one double per atom: the FP64 scratch of the index-order sums (SCR1).
  uint32_t* SURV = reinterpret_cast<uint32_t*>(A + ((b.max_n + 3) & ~3u));
  // per-step cross-pair list (alpha, beta, gamma) behind SCR1, then the sweep's FP64 pose X (3 per
  // atom, atom order) and exact per-atom samples ES
  float4* PL = reinterpret_cast<float4*>(SURV + 2 * ((b.max_n + 3) & ~3u));
  double* X = reinterpret_cast<double*>(PL + pair_cap<NS>());
  double* ES = X + 3 * ((b.max_n + 3) & ~3u);
  float* CF = reinterpret_cast<float*>(ES + ((b.max_n + 3) & ~3u));  // step cache: fixed-side sums
  double* BEST = reinterpret_cast<double*>(CF + 32);  // best candidate's moved-atom exact samples
  // pair state of the current pose (DFS space): CR[x * NS + w] = exact clash partners of atom x,
  // ZL = pairs whose exact margin is razor-thin, DINV = original index of DFS position x
  uint32_t* CR = reinterpret_cast<uint32_t*>(BEST + ((b.max_n + 3) & ~3u));
  uint32_t* AM = CR + NS * ((b.max_n + 3) & ~3u);  // pairs near the threshold, pending an FP64 verdict
  uint32_t* ZL = AM + NS * ((b.max_n + 3) & ~3u);  // + its counter at ZL[kZCap]
  uint32_t* DINV = ZL + kZCap + 4;
  double* SCR1 = reinterpret_cast<double*>(SURV);
  const CoarseGrid cg{cells,
                      0.5f * float(pk.cell_dims[0]),
                      0.5f * float(pk.cell_dims[1]),
                      0.5f * float(pk.cell_dims[2]),
                      pk.cell_dims[0],
                      pk.cell_dims[0] * pk.cell_dims[1],
                      0x4B000000u * (1u + pk.cell_dims[0] + pk.cell_dims[0] * pk.cell_dims[1]),
                      n_cells,
                      -pk.dz_bias};
  const uint32_t N = pr.n_restarts;
  const uint64_t total = uint64_t(b.n_lig) * N;
  const bool skip_inv = (pr.mode & GD_FLAG_SKIP_INVARIANT_CLASH) != 0;
  // per-warp counters (32-bit: a warp's share of one launch stays far below 2^32)
  uint32_t st_sexact = 0, st_sfall = 0, st_commit = 0, st_items = 0;
  // executed sweep work (the roofline's numerator counts only what ran): steps,
  // steps with an invariant clash, steps whose candidates were scored, moved-atom samples of the
  // scored candidates, and bump cross pairs (moved x fixed x candidates) of the steps that
  // evaluated them (none under an invariant clash: the reference's bump_check stops at its first
  // clashing pair, scoring.cpp:47-60). per-warp counters in shared memory (sweep_ctr,
  // plain adds by lane 0; registers here cost K1b spills, shared 64-bit atomics are CAS loops).
#ifdef GD_PHASE_TIMERS
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t_ph = clock64();
  int cur_ph = 7;
#endif

  for (;;) {
    uint32_t item = 0;
    if (lane == 0) item = atomicAdd(b.work_counter, 1u);
    item = __shfl_sync(FULL, item, 0);
    if (item >= total) break;
    if (*(volatile int*)b.error != 0) break;
    if (b.order) item = b.order[item];  // claims in start-target order (launch_dock)
    Item it;
    it.lig = item / N;
    it.rs = item - it.lig * N;
    it.m = b.meta[it.lig];
    it.n = it.m.n;
    if (it.n > 32u * NS || it.n <= b.fast_min_n) continue;  // another launch's ligand (mixed batch)
    ++st_items;
    GD_T(0);
    it.W = (it.n + 31) >> 5;
    const uint32_t n = it.n, R = it.m.nr;

    // ------------------------------------------------ the aligned pose (K1r: start pose, exact
    // alignment, apply_rotation_choice; docking.cpp:52-118) and its exact per-atom samples
    uint32_t pos[NS];
    double rad[NS];
    {
      const size_t base = size_t(it.m.atom_base) * N + size_t(it.rs) * n;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const uint32_t a = lane + 32 * s;
        rad[s] = a < n ? b.atoms[it.m.atom_base + a].w : 0.0;
        pos[s] = a < n ? b.dfs_pos[it.m.atom_base + a] : 0;
        if (a < n) {
          DINV[pos[s]] = a;
          X[3 * a] = b.rs_pose[3 * (base + a)];
          X[3 * a + 1] = b.rs_pose[3 * (base + a) + 1];
          X[3 * a + 2] = b.rs_pose[3 * (base + a) + 2];
          ES[a] = b.rs_es[base + a];
        }
      }
      __syncwarp();
    }
    // Position error bound (grid units, per axis) of every FP32 coordinate this item produces:
    // rounding of coordinates up to the grid size, plus the rotation error of the FP32 frames
    // (the dihedral axis from FP32 endpoints is good to ~1e-6 rad) times the ligand extent.
    // DESIGN.md §3.3 derives the constants.
    const float ext_g = b.rs_ext[item] * pk.inv_spacing_f;
    const float maxdim = float(max(pk.dims[0], max(pk.dims[1], pk.dims[2])));
    const float ptol = 1.5e-5f + 5e-7f * maxdim + 6e-6f * ext_g;
#if GD_K1B_FIELDF
    // coarse per-sample error bound (FP32 field in shared memory, else the quantised cells)
    const float eps_s = (SC ? pk.q_eps_f : pk.q_eps) + 3.0f * pk.max_step * ptol;
#else
    const float eps_s = pk.q_eps + 3.0f * pk.max_step * ptol;  // coarse per-sample error bound
#endif
    const float inv_n_scale = pk.coarse_scale / float(n);
    double score = b.rs_align_score[item];
    // restarts this kernel does not decide go to the FP64 kernel, which repeats them in the
    // reference's arithmetic throughout (launch_dock runs it after this kernel, on the same stream)
    bool abandoned = false;
    auto handoff = [&]() {
      if (lane == 0) b.slow_items[atomicAdd(b.slow_count, 1u)] = item;
      ++st_sfall;
      --st_items;
      abandoned = true;
    };
    // (the final pose and dihedrals are replayed by K2 from the decision trace)

    // ------------------------------------------------ dihedral sweep (docking.cpp:155-167, 197-215)
    // (non-tree layouts, whose moving sets are not DFS ranges, and S outside [2, 64] are the FP64
    // kernel's)
    if (R > 0 && pr.reps > 0 && pr.S > 0 && (!it.m.fast_ok || pr.S > 64 || pr.S < 2)) handoff();
    if (R > 0 && pr.reps > 0 && pr.S > 0 && !abandoned) {
      // Per-restart register caches (no global load on a step's critical path): lane r holds
      // rotamer r's bond (i | j << 16) and DFS range (s0 | e0 << 16, pos(i)) for r < 32 (later
      // rotamers load from global), and the FP32 half-angle (cos, sin) of its candidates k = lane + 1
      // (pass 0) and 33 + (lane >> lg2) (pass 1).
      uint32_t rc_ij = 0u, rc_se = 0u, rc_ip = 0u;
      if (lane < R) {
        const uint2 ij = b.rots[it.m.rot_base + lane];
        const ushort4 rd = b.rdfs[it.m.rot_base + lane];
        rc_ij = ij.x | (ij.y << 16);
        rc_se = uint32_t(rd.x) | (uint32_t(rd.y) << 16);
        rc_ip = rd.z;
      }
      const uint32_t n_cand_all = pr.S > 1 ? pr.S - 1 : 0;
      const uint32_t rem_all = n_cand_all > 32 ? n_cand_all - 32 : 0;
      const uint32_t lg2_all = rem_all <= 1 ? 5 : rem_all <= 2 ? 4 : rem_all <= 4 ? 3 : rem_all <= 8 ? 2 : rem_all <= 16 ? 1 : 0;
      const float2 cq_p0 = lane + 1 <= n_cand_all ? __ldg(pr.dtab_f + lane + 1) : make_float2(1.f, 0.f);
      const float2 cq_p1 = (lane >> lg2_all) < rem_all ? __ldg(pr.dtab_f + 33 + (lane >> lg2_all)) : make_float2(1.f, 0.f);
      // full-angle (cos, sin) of the same candidates, for the algebraic cross-pair margins
      const float2 cf_p0 = make_float2(fmaf(-2.f * cq_p0.y, cq_p0.y, 1.f), 2.f * cq_p0.x * cq_p0.y);
      // Per-pose caches, rebuilt after alignment and after every k != 0 commit:
      //   A[pos]     FP32 (gx, gy, gz, rho = cf*r/spacing) in DFS order,
      //   es, cs     exact FP64 and coarse per-atom samples, samb: coarse sample near a face,
      //   CR, ctot   exact clash partners of every atom (DFS bit rows, shared) and the number of
      //              clashing pairs, ZL / zcnt: pairs whose exact margin is razor-thin.
      float cs[NS];
      bool samb[NS];
      float rho[NS];
      float rmax = 0.f;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        rho[s] = float(__ddiv_rn(__dmul_rn(pr.clash, rad[s]), pk.spacing));
        if (lane + 32 * s < n) rmax = fmaxf(rmax, rho[s]);
      }
      rmax = warp_max(rmax);
      // |computed - exact| of d^2 - t^2 for pairs near the threshold (d ~ t <= 2 rmax):
      // 2 d |dd| with |dd| <= 2 sqrt(3) ptol, plus FP32 rounding of t^2 and the chain.
      const float tau = 16.0f * rmax * ptol + 4e-6f * rmax * rmax + 1e-6f;
      uint32_t ctot = 0u, zcnt = 0u;  // warp-uniform
      // Small ligands (NS <= GD_REG_ROWS_MAX_NS) keep the rows in registers instead: crow = exact
      // clash partners, arow = razor pairs (DFS bit rows of the lane's atoms), every row
      // recomputed at each refresh (measured faster there: one short loop per row word).
      constexpr bool kRegRows = NS <= GD_REG_ROWS_MAX_NS;
      uint32_t crow[NS][NS], arow[NS][NS];

      // (loops over the NS atom slots are not unrolled here: one copy of each body in the code,
      // register arrays indexed through pick/put selects)
      // all: every atom of the aligned pose; otherwise the atoms a k != 0 commit moved (mo in
      // original, md in DFS bit space). Only pairs with a moved atom change their distance, so only
      // their rows are recomputed: each moved atom's row from one ballot per word, and its bit in
      // every other atom's row by that atom's lane.
      auto refresh = [&](bool all, const uint32_t (&mo)[NS], const uint32_t (&md)[NS]) {
#pragma unroll 1
        for (int s = 0; s < NS; ++s) {
          const uint32_t a = lane + 32 * s;
          if (a < n && (all || ((pick<NS>(mo, s) >> lane) & 1u))) {
            const V3d pa{X[3 * a], X[3 * a + 1], X[3 * a + 2]};
            // FP32 grid coordinates (coarse path only: FP64 multiply by 1/spacing, error far
            // below the FP32 rounding that ptol covers)
            const float gx = float(__dmul_rn(__dsub_rn(pa.x, pk.origin[0]), pk.inv_spacing));
            const float gy = float(__dmul_rn(__dsub_rn(pa.y, pk.origin[1]), pk.inv_spacing));
            const float gz = float(__dmul_rn(__dsub_rn(pa.z, pk.origin[2]), pk.inv_spacing));
            A[pick<NS>(pos, s)] = make_float4(gx, gy, gz, pick<NS>(rho, s));
            float am = 1e30f;
#if GD_K1B_FIELDF
            float em_ = 1e30f;
            put<NS>(cs, s, SC ? sample_f<SC>(cgf, gx, gy, gz, am, em_) : coarse_sample(cg, gx, gy, gz, am));
#else
            put<NS>(cs, s, coarse_sample(cg, gx, gy, gz, am));
#endif
            put<NS>(samb, s, am <= ptol);
          }
        }
        __syncwarp();
        if constexpr (kRegRows) {
          bool any_amb = false;
#pragma unroll
          for (int s = 0; s < NS; ++s)
#pragma unroll
            for (int w = 0; w < NS; ++w) crow[s][w] = arow[s][w] = 0u;
#pragma unroll 1
          for (int s = 0; s < NS; ++s) {
            const uint32_t a = lane + 32 * s;
            if (a >= n) continue;
            const uint32_t ps = pick<NS>(pos, s);
            const float4 pa = A[ps];
            const uint32_t* adrow = b.adjd + it.m.adj_base + ps * it.W;
#pragma unroll 1
            for (int w = 0; w < NS; ++w) {
              if (uint32_t(w) >= it.W) break;
              // bonded partners and the atom itself are not bump pairs (scoring.cpp:53-55)
              const uint32_t skip = __ldg(adrow + w) | (ps >> 5 == uint32_t(w) ? 1u << (ps & 31) : 0u);
              const uint32_t qe = min(n, 32u * w + 32u);
              uint32_t cw = 0u, aw = 0u;
              for (uint32_t q = 32u * w; q < qe; ++q) {
                const float4 pb = A[q];
                const float dx = pa.x - pb.x, dy = pa.y - pb.y, dz = pa.z - pb.z;
                const float t = pa.w + pb.w;
                const float mg = fmaf(dx, dx, fmaf(dy, dy, fmaf(dz, dz, -t * t)));
                const uint32_t bit = 1u << (q & 31);
                cw |= mg < -tau ? bit : 0u;
                aw |= (mg >= -tau && mg <= tau) ? bit : 0u;
              }
              put2<NS>(crow, s, w, cw & ~skip);
              put2<NS>(arow, s, w, aw & ~skip);
              any_amb |= (aw & ~skip) != 0u;
            }
          }
          if (__any_sync(FULL, any_amb)) {  // near-threshold pairs: exact FP64 verdict
            for (uint32_t bb = 0; bb < n; ++bb) {
              const V3d pb{X[3 * bb], X[3 * bb + 1], X[3 * bb + 2]};
              const uint32_t q = b.dfs_pos[it.m.atom_base + bb];
              const double rb = b.atoms[it.m.atom_base + bb].w;
              const uint32_t bit = 1u << (q & 31), qw = q >> 5;
#pragma unroll
              for (int s = 0; s < NS; ++s) {
                const uint32_t aw = word_of<NS>(arow[s], qw);
                if (aw & bit) {
                  // exact verdict (clash iff d^2 < thr^2); the pair stays flagged ("razor") only
                  // if its exact margin is within 1e-8 A^2
                  const uint32_t a = lane + 32 * s;
                  const double mg = pair_margin_exact(V3d{X[3 * a], X[3 * a + 1], X[3 * a + 2]}, pb,
                                                      b.atoms[it.m.atom_base + a].w, rb, pr.clash);
                  const uint32_t set_c = mg < 0.0 ? bit : 0u, clr_a = fabs(mg) <= 1e-8 ? 0u : bit;
#pragma unroll
                  for (int w = 0; w < NS; ++w)
                    if (qw == uint32_t(w)) {
                      crow[s][w] |= set_c;
                      arow[s][w] &= ~clr_a;
                    }
                }
              }
            }
          }
        } else {
        // Rows in FP32 against tau; pairs within tau of the threshold are marked in AM (both rows)
        // and settled in FP64 by one pass below.
        uint32_t* zc = ZL + kZCap;  // razor-pair counter
        if (all) {
          // every row, lane-owned: each lane its atoms' rows, one word at a time against the
          // broadcast partners (the pair loop of bump_check, scoring.cpp:52-58)
          zcnt = 0u;
#pragma unroll 1
          for (int s = 0; s < NS; ++s) {
            if (lane + 32u * s >= n) continue;
            const uint32_t ps = pick<NS>(pos, s);
            const float4 pa = A[ps];
            const uint32_t* adrow = b.adjd + it.m.adj_base + ps * it.W;
#pragma unroll 1
            for (int w = 0; w < NS; ++w) {
              if (uint32_t(w) >= it.W) break;
              // bonded partners and the atom itself are not bump pairs (scoring.cpp:53-55)
              const uint32_t skip = __ldg(adrow + w) | (ps >> 5 == uint32_t(w) ? 1u << (ps & 31) : 0u);
              const uint32_t qe = min(n, 32u * w + 32u);
              uint32_t cw = 0u, aw = 0u;
              for (uint32_t q = 32u * w; q < qe; ++q) {
                const float4 pb = A[q];
                const float dx = pa.x - pb.x, dy = pa.y - pb.y, dz = pa.z - pb.z;
                const float t = pa.w + pb.w;
                const float mg = fmaf(dx, dx, fmaf(dy, dy, fmaf(dz, dz, -t * t)));
                const uint32_t bit = 1u << (q & 31);
                cw |= mg < -tau ? bit : 0u;
                aw |= (mg >= -tau && mg <= tau) ? bit : 0u;
              }
              CR[ps * NS + uint32_t(w)] = cw & ~skip;
              AM[ps * NS + uint32_t(w)] = aw & ~skip;
            }
          }
        } else {
          // after a commit: the rows of the moved atoms (one ballot per word), and their bits in
          // the partners' rows (by the partner's lane). Razor pairs with a moved atom leave the list.
          if (zcnt != 0u && zcnt <= kZCap) {
            const uint32_t e = lane < zcnt ? ZL[lane] : 0u;
            const bool keep = lane < zcnt && !bit4<NS>(md, e & 0xffffu) && !bit4<NS>(md, e >> 16);
            const uint32_t kb = __ballot_sync(FULL, keep);
            __syncwarp();
            if (keep) ZL[__popc(kb & ((1u << lane) - 1u))] = e;
            zcnt = __popc(kb);
          }
#pragma unroll 1
          for (int w0 = 0; w0 < NS; ++w0) {
            uint32_t bits = word_of<NS>(md, uint32_t(w0));
            while (bits) {
              const uint32_t p = 32u * uint32_t(w0) + uint32_t(__ffs(bits) - 1);
              bits &= bits - 1u;
              const float4 pp = A[p];
              const uint32_t pb = 1u << (p & 31);
#pragma unroll 1
              for (int t = 0; t < NS; ++t) {
                if (uint32_t(t) >= it.W) break;
                const uint32_t x = lane + 32u * uint32_t(t);
                const uint32_t bw = __ldg(b.adjd + it.m.adj_base + p * it.W + t);
                bool c = false, am = false;
                if (x < n && x != p && !((bw >> lane) & 1u)) {
                  const float4 px = A[x];
                  const float dx = pp.x - px.x, dy = pp.y - px.y, dz = pp.z - px.z;
                  const float tt = pp.w + px.w;
                  const float mg = fmaf(dx, dx, fmaf(dy, dy, fmaf(dz, dz, -tt * tt)));
                  c = mg < -tau;
                  am = mg >= -tau && mg <= tau;
                }
                const uint32_t wc = __ballot_sync(FULL, c), wa = __ballot_sync(FULL, am);
                if (lane == 0) {
                  CR[p * NS + uint32_t(t)] = wc;
                  AM[p * NS + uint32_t(t)] = wa;
                }
                if (x < n && x != p) {
                  uint32_t& rc = CR[x * NS + (p >> 5)];
                  rc = (rc & ~pb) | (c ? pb : 0u);
                  AM[x * NS + (p >> 5)] |= am ? pb : 0u;
                }
              }
              __syncwarp();
            }
          }
        }
        // near-threshold pairs: exact verdict (scoring.cpp:52-58: clash iff d^2 < thr^2), each pair
        // once (marked in both rows, settled from the lower one). A pair whose exact margin is
        // within 1e-8 A^2 is "razor": the FP64 rounding of a rotated candidate (~1e-12 A^2) could
        // flip it (ZL).
        if (lane == 0) *zc = zcnt;
        __syncwarp();
#pragma unroll 1
        for (int t = 0; t < NS; ++t) {
          const uint32_t x = lane + 32u * uint32_t(t);
          if (x >= n) continue;
#pragma unroll 1
          for (uint32_t w = 0; w < it.W; ++w) {
            uint32_t aw = AM[x * NS + w];
            if (GD_LIKELY(!aw)) continue;
            AM[x * NS + w] = 0u;
            aw &= ~range_word(w, 0u, x + 1u);  // partners above x
            while (aw) {
              const uint32_t q = 32u * w + uint32_t(__ffs(aw) - 1);
              aw &= aw - 1u;
              const uint32_t xo = DINV[x], qo = DINV[q];
              const double mgx = pair_margin_exact(V3d{X[3 * xo], X[3 * xo + 1], X[3 * xo + 2]},
                                                   V3d{X[3 * qo], X[3 * qo + 1], X[3 * qo + 2]},
                                                   b.atoms[it.m.atom_base + xo].w, b.atoms[it.m.atom_base + qo].w,
                                                   pr.clash);
              const uint32_t qb = 1u << (q & 31), xb = 1u << (x & 31);
              if (mgx < 0.0) {
                atomicOr(CR + x * NS + w, qb);
                atomicOr(CR + q * NS + (x >> 5), xb);
              } else {
                atomicAnd(CR + x * NS + w, ~qb);
                atomicAnd(CR + q * NS + (x >> 5), ~xb);
              }
              if (fabs(mgx) <= 1e-8) {
                const uint32_t at = atomicAdd(zc, 1u);
                if (at < kZCap) ZL[at] = x | (q << 16);
              }
            }
          }
        }
        __syncwarp();
        zcnt = *zc;
        uint32_t cnt = 0u;
#pragma unroll
        for (int t = 0; t < NS; ++t) {
          const uint32_t x = lane + 32u * uint32_t(t);
          if (x < n) {
#pragma unroll
            for (int w = 0; w < NS; ++w)
              if (uint32_t(w) < it.W) cnt += __popc(CR[x * NS + uint32_t(w)]);
          }
        }
        ctot = __reduce_add_sync(FULL, cnt) >> 1;  // every clashing pair sits in two rows
        }
      };
      // rotamer r's bond (i, j), DFS range (s0, e0) and DFS position of atom_i
      auto rot_info = [&](uint32_t rr, uint2& ij_, uint32_t& s0_, uint32_t& e0_, uint32_t& ip_) {
        if (rr < 32) {
          const uint32_t pij = __shfl_sync(FULL, rc_ij, rr), pse = __shfl_sync(FULL, rc_se, rr);
          ij_ = make_uint2(pij & 0xffffu, pij >> 16);
          s0_ = pse & 0xffffu;
          e0_ = pse >> 16;
          ip_ = __shfl_sync(FULL, rc_ip, rr);
        } else {
          ij_ = b.rots[it.m.rot_base + rr];
          const ushort4 rd = b.rdfs[it.m.rot_base + rr];
          s0_ = rd.x;
          e0_ = rd.y;
          ip_ = rd.z;
        }
      };
      // M' = moving set minus atom_j (molecule.cpp:166-169) of rotamer rr, in original (mo) and
      // DFS (md) bit spaces, and this lane's membership (inm). Fast layout: M' is the DFS range
      // (s0, e0), so both follow from the range.
      auto rot_masks = [&](uint32_t rr, uint2 ij_, uint32_t s0_, uint32_t e0_, uint32_t (&mo_)[NS],
                           uint32_t (&md_)[NS], bool (&inm_)[NS]) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          inm_[s] = lane + 32 * s < n && pos[s] > s0_ && pos[s] < e0_;
          mo_[s] = __ballot_sync(FULL, inm_[s]);  // slot s holds atoms 32 s + lane
          md_[s] = range_word(uint32_t(s), s0_ + 1, e0_);
        }
      };

      // The per-pose caches are rebuilt at ONE place, the top of the next step (one inlined copy
      // of refresh in the kernel's code): the aligned pose (all atoms) before the
      // first step, the atoms rotamer pend_r moved after a k != 0 commit.
      constexpr uint32_t kRefreshAll = 0xffffffffu, kRefreshNone = 0xfffffffeu;
      uint32_t pend_r = kRefreshAll;
      uint32_t vmask = 0u;  // step cache (rotamers r < 32): valid entries of CF
      for (uint32_t rep = 0; rep < pr.reps; ++rep) {
        for (uint32_t r = 0; r < R; ++r) {
          if (GD_UNLIKELY(pend_r != kRefreshNone)) {
            GD_T(3);
            uint32_t pmo[NS], pmd[NS];
            uint32_t ps0 = 0, pe0 = 0;
            if (pend_r == kRefreshAll) {
#pragma unroll
              for (int w = 0; w < NS; ++w) pmo[w] = pmd[w] = 0u;
            } else {
              uint2 pij;
              uint32_t pip;
              bool pinm[NS];
              rot_info(pend_r, pij, ps0, pe0, pip);
              rot_masks(pend_r, pij, ps0, pe0, pmo, pmd, pinm);
            }
            refresh(pend_r == kRefreshAll, pmo, pmd);
            pend_r = kRefreshNone;
          }
          GD_T(4);
          uint2 ij;
          uint32_t s0, e0, ipos;
          rot_info(r, ij, s0, e0, ipos);
          // M' = moving set minus atom_j (molecule.cpp:166-169), original (mo) and DFS (md) bit
          // spaces. Fast layout: M' is the DFS range (s0, e0), so both follow from the range.
          // Step cache: a rotamer whose last visit saw an invariant clash (fast layout, no razor
          // pairs) sees it again while the pose is unchanged (no k != 0 commit since), with the
          // same fixed-side sum (CF): its head is one shared load.
          uint32_t mo[NS], md[NS];
          bool inm[NS];
          bool inv, frag, elig0;
          float fsum = 0.f;
          // FP64 axis (rotate_fragment, molecule.cpp:150-160), computed when first needed; the
          // DegenerateAxisError check (len < 1e-12) only needs FP64 when the FP32 bond is tiny
          V3d pi{0, 0, 0}, axis{0, 0, 0};
          bool have_axis = false;
          auto get_axis = [&]() {
            if (have_axis) return;
            pi = V3d{X[3 * ij.x], X[3 * ij.x + 1], X[3 * ij.x + 2]};
            const V3d delta = vsub(V3d{X[3 * ij.y], X[3 * ij.y + 1], X[3 * ij.y + 2]}, pi);
            axis = vscale(__ddiv_rn(1.0, __dsqrt_rn(vdot(delta, delta))), delta);
            have_axis = true;
          };
          const bool cached = r < 32 && ((vmask >> r) & 1u);
          if (cached) {
            fsum = CF[r];
            inv = true;
            frag = elig0 = false;
#pragma unroll
            for (int s = 0; s < NS; ++s) {
              mo[s] = md[s] = 0u;
              inm[s] = false;
            }
          } else {
            rot_masks(r, ij, s0, e0, mo, md, inm);
            if constexpr (kRegRows) {
              bool inv_l = false, frag_l = false, cne_l = false;
#pragma unroll
              for (int s = 0; s < NS; ++s) {
                if (lane + 32 * s >= n) continue;
                // Invariant pairs: both in M', both outside M', and (m, atom_j) — j lies on the
                // axis, so |m - j| does not change with the angle either. Their exact verdicts
                // (crow) hold for every candidate unless the exact margin is razor-thin (arow).
                const bool isj = pos[s] == s0;
#pragma unroll
                for (int w = 0; w < NS; ++w) {
                  const uint32_t lo = 32u * w;
                  const uint32_t valid = lo + 32u <= n ? FULL : (lo >= n ? 0u : ((1u << (n - lo)) - 1u));
                  const uint32_t mdj = md[w] | ((s0 >> 5) == uint32_t(w) ? 1u << (s0 & 31) : 0u);
                  inv_l |= (crow[s][w] & (inm[s] ? mdj : isj ? valid : (~md[w] & valid))) != 0u;
                  if (inm[s]) frag_l |= (arow[s][w] & mdj) != 0u;
                  if (isj) frag_l |= (arow[s][w] & md[w]) != 0u;
                  cne_l |= crow[s][w] != 0u;
                }
                if (!inm[s]) fsum += cs[s];
              }
              inv = __any_sync(FULL, inv_l);
              frag = __any_sync(FULL, frag_l);
              elig0 = !__any_sync(FULL, cne_l);  // k = 0: the current pose passes bump_check
            } else {
            // Invariant pairs: both in M', both outside M', and (m, atom_j) — j lies on the axis, so
            // |m - j| does not change with the angle either. Their exact verdicts hold for every
            // candidate unless the exact margin is razor-thin (ZL). Of the pose's ctot clashing
            // pairs, `cross` have one atom in M' and the other outside M' + {j}: an invariant clash
            // exists iff ctot > cross, and k = 0 (the current pose) passes bump_check iff ctot == 0.
            uint32_t mj[NS];
#pragma unroll
            for (int w = 0; w < NS; ++w) mj[w] = md[w] | ((s0 >> 5) == uint32_t(w) ? 1u << (s0 & 31) : 0u);
            uint32_t cross = 0u;
#pragma unroll
            for (int t = 0; t < NS; ++t) {
              const uint32_t x = lane + 32u * uint32_t(t);
              if (x < n && ((md[t] >> lane) & 1u)) {
#pragma unroll
                for (int w = 0; w < NS; ++w)
                  if (uint32_t(w) < it.W) cross += __popc(CR[x * NS + uint32_t(w)] & ~mj[w]);
              }
            }
#pragma unroll
            for (int s = 0; s < NS; ++s)
              if (lane + 32 * s < n && !inm[s]) fsum += cs[s];
            inv = ctot > __reduce_add_sync(FULL, cross);
            elig0 = ctot == 0u;
            frag = zcnt > kZCap;
            if (GD_UNLIKELY(zcnt != 0u && !frag)) {  // a razor pair inside M' + {j}: its distance moves by rounding
              const uint32_t e = lane < zcnt ? ZL[lane] : 0u;
              frag = __any_sync(FULL, lane < zcnt && bit4<NS>(mj, e & 0xffffu) && bit4<NS>(mj, e >> 16));
            }
            }
            fsum = warp_sum(fsum);
            if (pr.S > 1) {
              const float4 fi = A[ipos], fj = A[s0];
              const float dx = fj.x - fi.x, dy = fj.y - fi.y, dz = fj.z - fi.z;
              if (GD_UNLIKELY(dx * dx + dy * dy + dz * dz < 1e-6f)) {
                const V3d qi{X[3 * ij.x], X[3 * ij.x + 1], X[3 * ij.x + 2]};
                const V3d delta = vsub(V3d{X[3 * ij.y], X[3 * ij.y + 1], X[3 * ij.y + 2]}, qi);
                if (__dsqrt_rn(vdot(delta, delta)) < 1e-12) {
                  if (lane == 0 && atomicCAS(b.error, 0, GD_ERR_DEGENERATE_AXIS) == 0) b.error[1] = int(b.lig_base + it.lig);
                  break;
                }
              }
            }
            if (r < 32 && inv && !frag) {  // warp-uniform
              if (lane == 0) CF[r] = fsum;
              __syncwarp();  // every lane reads CF[r] at a later step
              vmask |= 1u << r;
            }
          }
          {
            const uint32_t nm_c = e0 - s0 - 1;
            const uint32_t n_k = pr.S - 1;
            if (lane == 0) {
              uint32_t* c = sweep_ctr[warp];
              const bool scored = !(skip_inv && inv);
              c[0] += 1u;
              c[1] += inv ? 1u : 0u;
              c[2] += scored ? 1u : 0u;
              c[3] += scored ? nm_c * n_k : 0u;
              c[4] += scored && !inv ? nm_c * (n - nm_c - 1) * n_k : 0u;
            }
          }
          int32_t step_k = -1;
          const size_t trace_at = size_t(it.m.rot_base) * N * pr.reps + (size_t(it.rs) * pr.reps + rep) * R + r;
          bool committed = false;
          uint32_t bk = 0;
          double bs = 0.0;
          // the moved atoms' exact samples of the best candidate so far, from the scorer's scratch
          auto keep_best = [&]() {
#pragma unroll
            for (int t = 0; t < NS; ++t)
              if (inm[t]) BEST[lane + 32 * t] = SCR1[lane + 32 * t];
          };

          if (GD_UNLIKELY(frag)) {
            // a pair of the moving fragment within the razor margin of its bump threshold (its
            // FP64 distance moves by rounding under the rotation): the restart goes to the FP64
            // kernel, which repeats it in the reference's arithmetic throughout
            handoff();
            break;
          } else if (!(skip_inv && inv)) {
            GD_T(5);
            float res_s[2] = {-1e30f, -1e30f};
            uint32_t res_st[2] = {0u, 0u};
            // ---------------- coarse evaluation of every candidate k = 1 .. S-1 (faithful sweep).
            // With M' empty (atom_j a leaf: half the steps of the generated libraries) every
            // candidate is the current pose: no moved atom, no sample, no cross pair, and the
            // decision below needs none of the candidates' values.
            if (e0 > s0 + 1) {
            // pass-1 lanes per candidate: at most the moved atoms (no idle lanes to reduce over);
            // the candidates' half-angles move to that lane layout by one shuffle
            const uint32_t nm_s = e0 - s0 - 1;
            const uint32_t sh1 = min(lg2_all, nm_s <= 1 ? 0u : 32u - __clz(nm_s - 1u));
            const float2 cq1 = make_float2(__shfl_sync(FULL, cq_p1.x, min((lane >> sh1) << lg2_all, 31u)),
                                           __shfl_sync(FULL, cq_p1.y, min((lane >> sh1) << lg2_all, 31u)));
            const float2 cf1 = make_float2(fmaf(-2.f * cq1.y, cq1.y, 1.f), 2.f * cq1.x * cq1.y);
            const float4 fpi = A[ipos];
            const float4 fpj = A[s0];
            float ax = fpj.x - fpi.x, ay = fpj.y - fpi.y, az = fpj.z - fpi.z;
            {
              const float il = rsqrtf(fmaxf(ax * ax + ay * ay + az * az, 1e-30f));
              ax *= il;
              ay *= il;
              az *= il;
            }
            // Cross pairs. Rotating M' by theta about the unit axis a through pi
            // maps u = m - pi to h a + cos(theta) u_perp + sin(theta) (a x u), so for a fixed-side
            // atom f (w = f - pi) the bump margin of candidate k is
            //   d_k^2 - t^2 = alpha + beta cos(theta_k) + gamma sin(theta_k),
            //   alpha = (h_m - h_f)^2 + rho_m^2 + rho_f^2 - t^2, beta = -2 u_perp.w, gamma = -2 (a x u).w,
            // whose minimum over theta is (h_m - h_f)^2 + (rho_m - rho_f)^2 - t^2 (the distance to
            // the circle). A pair whose circle distance is >= t + 1e-3 grid units cannot clash at any
            // angle (the FP32 geometry is good to ~1e-5) and is dropped; the others go to the
            // per-warp list PL as (alpha, beta, gamma), which every candidate lane folds with two
            // FFMAs per pair (pairs with atom_j are invariant, see above). The list is folded
            // whenever the next moved atom's pairs might not fit.
            // With an invariant clash every candidate fails bump_check on that pair, where the
            // reference's bump_check returns (scoring.cpp:47-60 stops at the first clashing pair):
            // the cross pairs are not needed, only the candidates' scores (score_pose) are.
            float mmin0 = 1e30f, mmin1 = 1e30f;  // this lane's pass-0 candidate / pass-1 share
            float tau_a = 0.f;                     // tau plus the FP32 error of the algebraic form
            if (!inv) {
              float hq[NS], rq[NS], tq[NS], wx_[NS], wy_[NS], wz_[NS];
              float d2 = 0.f;
#pragma unroll
              for (int t = 0; t < NS; ++t) {
                const uint32_t q = lane + 32 * t;
                hq[t] = rq[t] = tq[t] = wx_[t] = wy_[t] = wz_[t] = 0.f;
                if (q < n) {
                  const float4 pq = A[q];
                  const float wx = pq.x - fpi.x, wy = pq.y - fpi.y, wz = pq.z - fpi.z;
                  const float h = fmaf(wx, ax, fmaf(wy, ay, wz * az));
                  wx_[t] = fmaf(-h, ax, wx);
                  wy_[t] = fmaf(-h, ay, wy);
                  wz_[t] = fmaf(-h, az, wz);
                  hq[t] = h;
                  rq[t] = sqrtf(fmaf(wx_[t], wx_[t], fmaf(wy_[t], wy_[t], wz_[t] * wz_[t])));
                  tq[t] = pq.w;
                  d2 = fmaxf(d2, fmaf(h, h, rq[t] * rq[t]));
                }
              }
              // |alpha|, |beta|, |gamma| <= 10 D^2 (D = largest distance from pi): FP32 rounding of
              // the terms and of the fold, the FP32 (cos, sin) and the non-unit FP32 axis, <= 8e-6 D^2
              tau_a = tau + 8e-6f * warp_max(d2);
              const uint32_t sub1 = lane & ((1u << sh1) - 1u), gs1 = 1u << sh1;
              uint32_t cnt = 0;
              auto fold = [&]() {
                __syncwarp();
                for (uint32_t e = 0; e < cnt; ++e) {
                  const float4 pe = PL[e];
                  mmin0 = fminf(mmin0, fmaf(pe.y, cf_p0.x, fmaf(pe.z, cf_p0.y, pe.x)));
                }
                for (uint32_t e = sub1; e < cnt; e += gs1) {
                  const float4 pe = PL[e];
                  mmin1 = fminf(mmin1, fmaf(pe.y, cf1.x, fmaf(pe.z, cf1.y, pe.x)));
                }
                __syncwarp();
                cnt = 0;
              };
              // one fold call site: before each moved atom when its pairs might not fit, and at the end
              for (uint32_t mq = s0 + 1;; ++mq) {
                if (mq >= e0 || cnt + 32u * NS > pair_cap<NS>()) fold();
                if (mq >= e0) break;
                const float4 pm = A[mq];
                const float ux = pm.x - fpi.x, uy = pm.y - fpi.y, uz = pm.z - fpi.z;
                const float hm = fmaf(ux, ax, fmaf(uy, ay, uz * az));
                const float upx = fmaf(-hm, ax, ux), upy = fmaf(-hm, ay, uy), upz = fmaf(-hm, az, uz);
                const float rm2 = fmaf(upx, upx, fmaf(upy, upy, upz * upz)), rm = sqrtf(rm2);
                const float vx = fmaf(ay, uz, -az * uy), vy = fmaf(az, ux, -ax * uz), vz = fmaf(ax, uy, -ay * ux);
#pragma unroll
                for (int t = 0; t < NS; ++t) {
                  const uint32_t q = lane + 32 * t;
                  const bool fixed = q < n && (q < s0 || q >= e0);
                  const float dh = hq[t] - hm, dr = rq[t] - rm, tt = tq[t] + pm.w, T = tt + 1e-3f;
                  const bool surv = fixed && fmaf(dh, dh, dr * dr) < T * T;
                  const uint32_t ball = __ballot_sync(FULL, surv);
                  if (surv) {
                    const float al = fmaf(dh, dh, fmaf(rq[t], rq[t], fmaf(-tt, tt, rm2)));
                    const float be = -2.0f * fmaf(upx, wx_[t], fmaf(upy, wy_[t], upz * wz_[t]));
                    const float ga = -2.0f * fmaf(vx, wx_[t], fmaf(vy, wy_[t], vz * wz_[t]));
                    PL[cnt + __popc(ball & ((1u << lane) - 1u))] = make_float4(al, be, ga, 0.f);
                  }
                  cnt += __popc(ball);
                }
              }
            }
            const uint32_t n_cand = pr.S - 1;  // k = 1 .. S-1
            const uint32_t rem = n_cand > 32 ? n_cand - 32 : 0;
            const uint32_t lg2 = sh1;
#pragma unroll 1
            for (int pass = 0; pass < 2; ++pass) {
              if (pass == 1 && rem == 0) break;
              const uint32_t sh = pass == 0 ? 0u : lg2;  // log2 of lanes per candidate
              const uint32_t gs = 1u << sh;
              const uint32_t grp = lane >> sh, sub = lane & (gs - 1);
              const uint32_t k = pass == 0 ? lane + 1 : 33 + grp;
              const bool active = pass == 0 ? (k <= n_cand) : (grp < rem);
              float part = 0.f, amin = 1e30f, emin = 1e30f;
              float mmin = pass == 0 ? mmin0 : mmin1;
              if (active) {
                // moved-atom samples at this lane's angle: the rotation matrix of the half-angle
                // quaternion (about_axis, geometry.hpp:46-50) in FP32
                const float2 cq = pass == 0 ? cq_p0 : cq1;
                const float qw = cq.x, qx = ax * cq.y, qy = ay * cq.y, qz = az * cq.y;
                const float xx = qx * qx, yy = qy * qy, zz = qz * qz, xy = qx * qy, xz = qx * qz, yz = qy * qz;
                const float wx = qw * qx, wy = qw * qy, wz = qw * qz;
                const float m00 = 1.f - 2.f * (yy + zz), m01 = 2.f * (xy - wz), m02 = 2.f * (xz + wy);
                const float m10 = 2.f * (xy + wz), m11 = 1.f - 2.f * (xx + zz), m12 = 2.f * (yz - wx);
                const float m20 = 2.f * (xz - wy), m21 = 2.f * (yz + wx), m22 = 1.f - 2.f * (xx + yy);
                const float tvx = fpi.x - fmaf(m00, fpi.x, fmaf(m01, fpi.y, m02 * fpi.z));
                const float tvy = fpi.y - fmaf(m10, fpi.x, fmaf(m11, fpi.y, m12 * fpi.z));
                const float tvz = fpi.z - fmaf(m20, fpi.x, fmaf(m21, fpi.y, m22 * fpi.z));
                for (uint32_t mq = s0 + 1 + sub; mq < e0; mq += gs) {
                  const float4 pm = A[mq];
                  const float gx = fmaf(m00, pm.x, fmaf(m01, pm.y, fmaf(m02, pm.z, tvx)));
                  const float gy = fmaf(m10, pm.x, fmaf(m11, pm.y, fmaf(m12, pm.z, tvy)));
                  const float gz = fmaf(m20, pm.x, fmaf(m21, pm.y, fmaf(m22, pm.z, tvz)));
#if GD_K1B_FIELDF
                  // (a field too large for shared memory: the quantised cells through L1/L2 are faster)
                  part += SC ? sample_f<SC>(cgf, gx, gy, gz, amin, emin) : coarse_sample_e(cg, gx, gy, gz, amin, emin);
#else
                  part += coarse_sample_e(cg, gx, gy, gz, amin, emin);
#endif
                }
              }
              for (uint32_t o = 1; o < gs; o <<= 1) {  // group reduction (pass 2)
                part += __shfl_xor_sync(FULL, part, o);
                amin = fminf(amin, __shfl_xor_sync(FULL, amin, o));
                mmin = fminf(mmin, __shfl_xor_sync(FULL, mmin, o));
                emin = fminf(emin, __shfl_xor_sync(FULL, emin, o));
              }
              uint32_t st = 0;
              if (active) {
                st = mmin < -tau_a ? ST_CLASH : (mmin >= tau_a ? ST_OK : ST_XAMB);
                if (amin <= ptol) st |= ST_SAMB;
                if (emin > ptol) st |= ST_ALLOUT;
              }
              const float sc = (fsum + part) * inv_n_scale;
              if (pass == 0) {
                res_s[0] = sc;
                res_st[0] = st;
              } else {
                const float s2 = __shfl_sync(FULL, sc, (lane << sh) & 31);
                const uint32_t t2 = __shfl_sync(FULL, st, (lane << sh) & 31);
                if (lane < rem) {
                  res_s[1] = s2;
                  res_st[1] = t2;
                }
              }
            }
            }

            GD_T(6);
            // ---------------- exact decisions (reference semantics, docking.cpp:131-147)
            if (!inv && s0 + 1 >= e0) {
              // M' empty (atom_j is a leaf): every candidate is the current pose, so k = 0 wins
              // whenever it is eligible (lowest k on the exact tie) and nothing else can
              committed = elig0;
              bk = 0;
              bs = score;
            } else if (!inv) {
              // Both passes' candidates go through one loop (bit 32 h + lane: pass h, lane's k),
              // so each exact path below exists once in the kernel's code (instruction-cache
              // footprint of the step), in ascending k.
              {  // cross pairs within tau of the threshold: exact
                unsigned long long pend = __ballot_sync(FULL, (res_st[0] & ST_XAMB) != 0u) |
                                          (uint64_t(__ballot_sync(FULL, (res_st[1] & ST_XAMB) != 0u)) << 32);
                while (GD_UNLIKELY(pend != 0ull)) {
                  const uint32_t bit = uint32_t(__ffsll(static_cast<long long>(pend)) - 1);
                  pend &= pend - 1;
                  const uint32_t src = bit & 31u, h = bit >> 5;
                  const uint32_t k = (h == 0 ? 1u : 33u) + src;
                  ++st_sexact;
                  if (lane == 0) sweep_ctr[warp][9] += 1u;
                  get_axis();
                  const bool cl = exact_clash_g<NS>(b, it.m.atom_base, it.m.adj_base, n, X, GD_MO4(mo), true, pi,
                                                    frag_quat(pr.dtab[k], axis), pr.clash, true, lane);
                  const uint32_t nst = cl ? ST_CLASH : ST_OK;
                  if (lane == src) {
                    if (h == 0) res_st[0] = (res_st[0] & (ST_SAMB | ST_ALLOUT)) | nst;
                    else res_st[1] = (res_st[1] & (ST_SAMB | ST_ALLOUT)) | nst;
                  }
                }
              }
              // Relative screening: all candidates share the fixed atoms (same coarse and exact
              // values), so two candidates' exact scores differ from their coarse difference by at
              // most the moved atoms' error: 2 * eps_rel with eps_rel = |M'| eps_sample / n.
              const uint32_t nm = e0 - s0 - 1;
              const float eps_rel =
                  (float(nm) * (eps_s + 3e-6f) + 6e-8f * (float(nm) * float(nm) + float(n))) / float(n) + 2e-7f;
              // k = 0 in the same coarse terms: fixed part + the cached coarse values of M'
              float p0 = 0.f;
              bool samb0 = false;
#pragma unroll
              for (int s = 0; s < NS; ++s)
                if (inm[s]) {
                  p0 += cs[s];
                  samb0 |= samb[s];
                }
              p0 = warp_sum(p0);
              samb0 = __any_sync(FULL, samb0);
              float Bl = (elig0 && !samb0) ? (fsum + p0) * inv_n_scale : -1e30f;
#pragma unroll
              for (int h = 0; h < 2; ++h)
                if ((res_st[h] & ST_OK) && !(res_st[h] & ST_SAMB)) Bl = fmaxf(Bl, res_s[h]);
              Bl = warp_max(Bl);
              const float thr_k = Bl - 2.0f * eps_rel;
              if (elig0) {  // k = 0: the current pose, score_pose(current) == the carried score
                committed = true;
                bk = 0;
                bs = score;
              }
              bool allout_done = false;  // candidates with every moved atom clearly outside tie exactly
              {
                const bool need0 = (res_st[0] & ST_OK) && ((res_st[0] & ST_SAMB) || res_s[0] >= thr_k);
                const bool need1 = (res_st[1] & ST_OK) && ((res_st[1] & ST_SAMB) || res_s[1] >= thr_k);
                unsigned long long pend = __ballot_sync(FULL, need0) | (uint64_t(__ballot_sync(FULL, need1)) << 32);
                const unsigned long long allout = __ballot_sync(FULL, (res_st[0] & ST_ALLOUT) != 0u) |
                                                  (uint64_t(__ballot_sync(FULL, (res_st[1] & ST_ALLOUT) != 0u)) << 32);
                while (GD_UNLIKELY(pend != 0ull)) {
                  const uint32_t bit = uint32_t(__ffsll(static_cast<long long>(pend)) - 1);
                  pend &= pend - 1;
                  if ((allout >> bit) & 1ull) {
                    if (allout_done) continue;
                    allout_done = true;
                  }
                  const uint32_t k = ((bit >> 5) == 0 ? 1u : 33u) + (bit & 31u);
                  ++st_sexact;
                  const uint32_t stk = __shfl_sync(FULL, (bit >> 5) == 0 ? res_st[0] : res_st[1], bit & 31u);
                  if (lane == 0) sweep_ctr[warp][((allout >> bit) & 1ull) ? 7 : (stk & ST_SAMB) ? 8 : 6] += 1u;
                  get_axis();
                  const double sk = exact_candidate_score_g<NS>(pk, n, X, ES, GD_MO4(mo), true, pi,
                                                                frag_quat(pr.dtab[k], axis), lane, SCR1);
                  if (!committed || sk > bs || (sk == bs && k < bk)) {
                    committed = true;
                    bk = k;
                    bs = sk;
                    keep_best();
                  }
                }
              }
            }
          }
          if (committed) {
            step_k = int32_t(bk);
            score = bs;
            ++st_commit;
            if (GD_UNLIKELY(bk != 0)) {  // commit = rotate_fragment(current, r, k*delta), FP64
              get_axis();
              const double4 dt = pr.dtab[bk];
              const Qd q = frag_quat(dt, axis);
#pragma unroll
              for (int s = 0; s < NS; ++s)
                if (inm[s]) {
                  const uint32_t a = lane + 32 * s;
                  const V3d v = rotated_about(V3d{X[3 * a], X[3 * a + 1], X[3 * a + 2]}, pi, q);
                  X[3 * a] = v.x;
                  X[3 * a + 1] = v.y;
                  X[3 * a + 2] = v.z;
                  // the exact sample of the new position: computed (bit for bit: same FP64
                  // rotation, same sampler) when candidate bk was scored exactly
                  ES[a] = BEST[a];
                }
              __syncwarp();
              pend_r = r;  // the caches of the moved atoms are rebuilt at the top of the next step
              if (lane == 0) sweep_ctr[warp][5] += 1u;
              vmask = 0u;  // the pose changed: every cached step head is stale
            }
          }
          if (lane == 0) b.rs_step_k[trace_at] = step_k;
        }
        if (abandoned || *(volatile int*)b.error != 0) break;
      }
    }
    if (*(volatile int*)b.error != 0) break;
    if (abandoned) continue;
    GD_T(7);
    // ------------------------------------------------ restart result (K2 replays its pose)
    if (lane == 0) {
      b.rs_score[item] = score;
      uint32_t* c = sweep_ctr[warp];
      if ((c[3] | c[4]) >= 0x80000000u) {  // keep the 32-bit per-warp counters far from wrapping
        for (int i = 0; i < int(kSweepCtr); ++i) {
          atomicAdd(b.stats + 16 + i, (unsigned long long)c[i]);
          c[i] = 0u;
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    atomicAdd(b.stats + 0, (unsigned long long)st_items);
    atomicAdd(b.stats + 3, (unsigned long long)st_sexact);
    atomicAdd(b.stats + 4, (unsigned long long)st_sfall);
    atomicAdd(b.stats + 5, (unsigned long long)st_commit);
#ifdef GD_PHASE_TIMERS
    GD_T(7);
    for (int i = 0; i < 8; ++i) atomicAdd(b.stats + 8 + i, (unsigned long long)ph[i]);
#endif
  }
  __syncthreads();
  if (threadIdx.x < kSweepCtr) {
    unsigned long long t = 0ull;
    for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) t += sweep_ctr[w][threadIdx.x];
    atomicAdd(b.stats + 16 + threadIdx.x, t);
  }
}

// Shared-memory plan of one persistent kernel: the pocket cells (when they fit next to 8 warp
// slots) plus one slot per warp, as many warps as fit up to NT / 32.
struct SmemPlan {
  bool cells_in_smem;
  int warps;
  size_t smem;
};

// min_warps_sc: the cells go to shared memory only if at least this many warp slots still fit
// beside them (K1a: 8, its gathers are the hot path; K1b: 12, its few samples can come from L1/L2
// while more resident warps hide the sweep's latency).
// `reserve`: the kernel's static shared memory (K1b's DevPocket copy)
static SmemPlan plan_smem(const DevPocket& pk, size_t slot_bytes, int max_warps, int min_warps_sc,
                          size_t reserve = 0) {
  const uint32_t n_cells = pk.cell_dims[0] * pk.cell_dims[1] * pk.cell_dims[2];
  const size_t cell_bytes = size_t(n_cells + 1) * sizeof(uint4);  // + the dummy cell
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  optin -= int(reserve);
  SmemPlan p{};
  p.cells_in_smem = cell_bytes + size_t(min_warps_sc) * slot_bytes <= size_t(optin);
  const size_t avail = size_t(optin) - (p.cells_in_smem ? cell_bytes : 0);
  p.warps = int(avail / slot_bytes);
  if (p.warps > max_warps) p.warps = max_warps;
  p.smem = (p.cells_in_smem ? cell_bytes : 0) + slot_bytes * size_t(p.warps > 0 ? p.warps : 0);
  return p;
}

template <class K>
static cudaError_t launch_persistent(K kernel, const SmemPlan& p, int n_sms, cudaStream_t stream, const DevPocket& pk,
                                     const DevParams& pr, const DevBatch& b, uint32_t slot_floats) {
  if (p.warps < 1) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p.smem));
  if (e != cudaSuccess) return e;
  kernel<<<n_sms, 32 * p.warps, p.smem, stream>>>(pk, pr, b, slot_floats);
  return cudaGetLastError();
}

// K1a (coarse alignment, NTA threads) then K1b (exact refinement + dihedral sweep, NTB threads).
template <int NS, int NTA, int NTB>
static cudaError_t launch_ns(const DevPocket& pk, const DevParams& pr, const DevBatch& b, int n_sms,
                             cudaStream_t stream, cudaEvent_t mid, cudaStream_t stream_b) {
  const uint32_t npad_max = (b.max_n + 3) & ~3u;
  const uint32_t slot_a = 4 * npad_max;                    // A (float4 per atom)
  // A (4 floats/atom) + SCR1 (1 double/atom) + PL + X (3 doubles/atom) + ES (1 double/atom)
  // + CR and BR (NS words per atom each) + ZL (+ counter) + DINV
  const uint32_t slot_b = 6 * npad_max + 4 * pair_cap<NS>() + 8 * npad_max + 32 + 2 * npad_max + 2 * NS * npad_max +
                          kZCap + 4 + npad_max;
  const SmemPlan pa = plan_smem(pk, slot_a * sizeof(float), NTA / 32, 8);
  // cells in shared memory: 12 / 14 / 12 warps for NS = 1 / 2 / 4 (GD_ALIGN_THREADS_NS1, GD_ALIGN_THREADS,
  // GD_ALIGN_THREADS_NS4); cells through L1 (large
  // grids): 16 warps x 128 (GD_ALIGN_THREADS_L1)
  const SmemPlan pg = plan_smem(pk, slot_a * sizeof(float), GD_ALIGN_THREADS_L1 / 32, 8);
  cudaError_t e =
      pa.cells_in_smem
          ? launch_persistent(align_coarse_kernel<NS, NTA, true>, pa, n_sms, stream, pk, pr, b, slot_a)
          : launch_persistent(align_coarse_kernel<NS, GD_ALIGN_THREADS_L1, false>, pg, n_sms, stream, pk, pr, b, slot_a);
  if (e != cudaSuccess) return e;
  if (mid && (e = cudaEventRecord(mid, stream)) != cudaSuccess) return e;
  if (stream_b && stream_b != stream) {  // K1b on its own stream, after this batch's K1a
    if ((e = cudaStreamWaitEvent(stream_b, mid, 0)) != cudaSuccess) return e;
    stream = stream_b;
  }
  // K1r (exact alignment): 3 n doubles of pose + 3 n of scratch per warp, FP64 field in shared
  // memory when it fits. Small ligands with the field in shared memory: 32 warps (C2 K1r -22 %);
  // otherwise 16 (with the field from L2, 32 warps were slower: C5 +5 %).
  {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const uint32_t slot_r = 6 * npad_max;
    const size_t fbytes = size_t(pk.dims[0]) * pk.dims[1] * pk.dims[2] * sizeof(double);
    auto launch_r = [&](auto kr, int nt) -> bool {  // false: the field does not fit beside nt threads
      size_t smem_r = size_t(slot_r) * sizeof(double) * size_t(nt / 32);
      const uint32_t fs_r = smem_r + fbytes + 1024 <= size_t(optin) ? 1u : 0u;
      if (!fs_r && nt != GD_REFINE_THREADS_NS4) return false;
      if (fs_r) smem_r += fbytes;
      if ((e = cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_r))) != cudaSuccess)
        return true;
      kr<<<n_sms, nt, smem_r, stream>>>(pk, pr, b, slot_r, fs_r);
      e = cudaGetLastError();
      return true;
    };
    if (!(NS <= 2 && launch_r(align_refine_kernel<NS, GD_REFINE_THREADS>, GD_REFINE_THREADS)))
      launch_r(align_refine_kernel<NS, GD_REFINE_THREADS_NS4>, GD_REFINE_THREADS_NS4);
    if (e != cudaSuccess) return e;
  }
  constexpr size_t kK1bStatic = 2048;  // the kernel's __shared__ DevPocket + per-warp counters, rounded up
#if GD_K1B_FIELDF
  SmemPlan pb{};
  {  // the warps' slots, then the FP32 field if it fits beside NTB / 32 of them (SC)
    int dv = 0, oi = 0;
    cudaGetDevice(&dv);
    cudaDeviceGetAttribute(&oi, cudaDevAttrMaxSharedMemoryPerBlockOptin, dv);
    const size_t avail = size_t(oi) - kK1bStatic, slot_bytes = slot_b * sizeof(float);
    const size_t ff_bytes = size_t((pk.f_count + 3u) & ~3u) * sizeof(float);
    pb.warps = int(std::min<size_t>(NTB / 32, avail / slot_bytes));
    pb.cells_in_smem = size_t(pb.warps) * slot_bytes + ff_bytes <= avail;
    pb.smem = size_t(pb.warps) * slot_bytes + (pb.cells_in_smem ? ff_bytes : 0);
  }
#else
  SmemPlan pb = plan_smem(pk, slot_b * sizeof(float), NTB / 32, GD_K1B_MIN_WARPS_SC, kK1bStatic);
#endif
  if (pb.warps < 1) return cudaErrorInvalidConfiguration;
  // the FP64 field goes to shared memory too when it fits beside the slots (24^3: 110 KB)
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t field_bytes = size_t(pk.dims[0]) * pk.dims[1] * pk.dims[2] * sizeof(double);
#ifndef GD_K1B_FIELD_SMEM
#define GD_K1B_FIELD_SMEM 1
#endif
  const uint32_t fs = GD_K1B_FIELD_SMEM && pb.smem + field_bytes + kK1bStatic <= size_t(optin) ? 1u : 0u;
  if (fs) pb.smem += field_bytes;
  auto kb = pb.cells_in_smem ? dock_fast_kernel<NS, NTB, true> : dock_fast_kernel<NS, NTB, false>;
  e = cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pb.smem));
  if (e != cudaSuccess) return e;
  kb<<<n_sms, 32 * pb.warps, pb.smem, stream>>>(pk, pr, b, slot_b, fs);
  return cudaGetLastError();
}

cudaError_t launch_fast(const DevPocket& pk, const DevParams& pr, const DevBatch& b, int n_sms,
                        cudaStream_t stream, cudaEvent_t mid, cudaStream_t stream_b) {
  if (b.max_n <= 32) return launch_ns<1, GD_ALIGN_THREADS_NS1, GD_FAST_THREADS>(pk, pr, b, n_sms, stream, mid, stream_b);
  if (b.max_n <= 64) return launch_ns<2, GD_ALIGN_THREADS, GD_FAST_THREADS>(pk, pr, b, n_sms, stream, mid, stream_b);
  if (b.max_n <= 128)
    return launch_ns<4, GD_ALIGN_THREADS_NS4, GD_FAST_THREADS_NS4>(pk, pr, b, n_sms, stream, mid, stream_b);
  return cudaErrorNotSupported;  // launch_dock routes > 128 atoms to the exact kernel
}

cudaError_t launch_align_big(const DevPocket& pk, const DevParams& pr, const DevBatch& b, int n_sms,
                             cudaStream_t stream) {
  // (ligands beyond kAlignBigMaxAtoms are skipped by the kernel: the FP64 kernel aligns them)
  const uint32_t slot_a = 4 * ((std::min(b.max_n, kAlignBigMaxAtoms) + 3) & ~3u);
  const SmemPlan pa = plan_smem(pk, slot_a * sizeof(float), GD_ALIGN_THREADS_NS4 / 32, 8);
  const SmemPlan pg = plan_smem(pk, slot_a * sizeof(float), GD_ALIGN_THREADS_L1 / 32, 8);
  return pa.cells_in_smem
             ? launch_persistent(align_coarse_kernel<8, GD_ALIGN_THREADS_NS4, true>, pa, n_sms, stream, pk, pr, b, slot_a)
             : launch_persistent(align_coarse_kernel<8, GD_ALIGN_THREADS_L1, false>, pg, n_sms, stream, pk, pr, b,
                                 slot_a);
}

uint32_t k1a_qt_groups() { return uint32_t(kQtGroups); }

bool k1a_cells_in_smem(const DevPocket& pk, uint32_t max_n) {
  const uint32_t npad = (std::min(max_n, kFastMaxAtoms) + 3) & ~3u;
  return plan_smem(pk, 4 * npad * sizeof(float), GD_ALIGN_THREADS / 32, 8).cells_in_smem;
}

}  // namespace gdk
