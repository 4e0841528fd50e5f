// GeoDock pose search on sm_100a: kernels and launchers.
//
//   K1  dock_*_kernel   persistent CTAs (one per SM); every warp repeatedly claims one
//                       (ligand, restart) work item from a global counter and runs the reference's
//                       per-restart search on it: start pose (docking.cpp:52-69) -> exhaustive rigid
//                       alignment (:71-91, :110-118) -> reps x rotamers dihedral sweep (:127-167).
//   K2  finalize_kernel warp per ligand: best restart by strict > (lowest id on ties,
//                       docking.cpp:216) and copy of its pose / dihedrals into the result arrays.
//   K3  top-k           device radix sort of (score, ligand) -> first k records.
//
// Two K1 variants share this file: dock_exact_kernel (FP64 everywhere, the reference's arithmetic)
// and dock_fast_kernel (gd_fast.cuh: FP32 coarse screen + FP64 refinement). DESIGN.md §3.
#include <cub/cub.cuh>

#include <algorithm>

#include "gd_exact.cuh"
#include "gd_fast.cuh"
#include "gd_internal.h"

namespace gdk {

namespace {

__device__ __forceinline__ void raise_error(const DevBatch& b, int code, uint32_t lig) {
  if (atomicCAS(b.error, 0, code) == 0) b.error[1] = int(b.lig_base + lig);  // library index
}

__device__ __forceinline__ bool bit_of(const uint32_t* words, uint32_t a) {
  return (__ldg(words + (a >> 5)) >> (a & 31)) & 1u;
}

// centroid (geometry.cpp:40-46): index-order sum then * (1/n). Every lane computes it redundantly
// from shared memory so no shuffle reduction (which would reorder the sum) is needed.
__device__ __forceinline__ V3d centroid_smem(const double* P, uint32_t n) {
  V3d s{0.0, 0.0, 0.0};
  for (uint32_t a = 0; a < n; ++a) s = vadd(s, V3d{P[3 * a], P[3 * a + 1], P[3 * a + 2]});
  return vscale(__ddiv_rn(1.0, double(n)), s);
}

__device__ __forceinline__ V3d ld3(const double* P, uint32_t a) {
  return V3d{P[3 * a], P[3 * a + 1], P[3 * a + 2]};
}
__device__ __forceinline__ void st3(double* P, uint32_t a, V3d v) {
  P[3 * a] = v.x;
  P[3 * a + 1] = v.y;
  P[3 * a + 2] = v.z;
}

}  // namespace

// --------------------------------------------------------------------------------------------
// K1 exact: the reference algorithm in FP64, warp-parallel but with the reference's summation
// orders. Shared memory per warp: pose P[3n], candidate C[3n], samples S[n] (doubles).
// --------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024, 1)
    dock_exact_kernel(DevPocket pk, DevParams pr, DevBatch b, uint32_t smem_stride, uint32_t min_n,
                      uint32_t list_mode) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = threadIdx.x >> 5;
  double* P = reinterpret_cast<double*>(smem_raw) + size_t(warp) * smem_stride;
  const uint32_t nmax = b.max_n;
  double* Cd = P + 3 * nmax;
  double* S = Cd + 3 * nmax;
  const uint32_t N = pr.n_restarts;
  const uint64_t total = uint64_t(b.n_lig) * N;

  // list mode: the restarts the fast sweep handed over (b.slow_items, b.slow_count of them)
  const uint32_t n_list = list_mode ? *(volatile unsigned int*)b.slow_count : 0u;
  for (;;) {
    uint32_t item = 0;
    if (lane == 0) item = atomicAdd(b.work_counter, 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (list_mode) {
      if (item >= n_list) break;
      item = b.slow_items[item];
    } else if (item >= total) {
      break;
    }
    if (*(volatile int*)b.error != 0) break;
    const uint32_t lig = item / N;
    const uint32_t rs = item - lig * N;
    const LigMeta m = b.meta[lig];
    const uint32_t n = m.n, R = m.nr, W = (n + 31) >> 5;
    if (!list_mode && n < min_n) continue;  // mixed batch: the fast kernels' ligand
    // min_n > 0 (or list mode): K1a ran for these ligands; its candidate list (ncand >= 0) contains
    // every rotation that can be the exact argmax
    // (ligands beyond kAlignBigMaxAtoms had no K1a: every rotation in FP64)
    const int32_t ncand = (list_mode || min_n > 0) && n <= kAlignBigMaxAtoms ? b.rs_ncand[item] : -1;

    // ---- starting pose (docking.cpp:52-69); q and target come from the host packer (libm).
    for (uint32_t a = lane; a < n; a += 32) {
      const double4 at = b.atoms[m.atom_base + a];
      st3(P, a, V3d{at.x, at.y, at.z});
    }
    __syncwarp();
    const V3d c0 = centroid_smem(P, n);
    const double4 q4 = b.start[2 * size_t(item)];
    const double4 t4 = b.start[2 * size_t(item) + 1];
    const Qd qs{q4.x, q4.y, q4.z, q4.w};
    const V3d tgt{t4.x, t4.y, t4.z};
    __syncwarp();
    for (uint32_t a = lane; a < n; a += 32) st3(P, a, vadd(qapply(qs, vsub(ld3(P, a), c0)), tgt));
    __syncwarp();

    // ---- exhaustive alignment (best_rotation_in_range, docking.cpp:71-91)
    const V3d c = centroid_smem(P, n);
    double best_s = -1.0;
    uint32_t best_g = 0xffffffffu;
    const uint32_t n_eval = ncand >= 0 ? uint32_t(ncand) : pr.G;
    for (uint32_t ci = lane; ci < n_eval; ci += 32) {
      const uint32_t g = ncand >= 0 ? uint32_t(b.rs_cand[size_t(item) * kAlignCand + ci]) : ci;
      const double4 gq = pr.grid[g];
      const Qd q{gq.x, gq.y, gq.z, gq.w};
      double sum = 0.0;
      for (uint32_t a = 0; a < n; ++a) sum = __dadd_rn(sum, sample_exact(pk, rotated_about(ld3(P, a), c, q)));
      const double s = __ddiv_rn(sum, double(n));
      if (best_g == 0xffffffffu || s > best_s || (s == best_s && g < best_g)) {
        best_s = s;
        best_g = g;
      }
    }
    // combine (docking.cpp:93-108): higher score wins, equal -> lower index.
    for (int off = 16; off > 0; off >>= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, best_s, off);
      const uint32_t og = __shfl_xor_sync(0xffffffffu, best_g, off);
      const bool take = og != 0xffffffffu &&
                        (best_g == 0xffffffffu || os > best_s || (os == best_s && og < best_g));
      if (take) {
        best_s = os;
        best_g = og;
      }
    }
    // apply_rotation_choice (docking.cpp:110-118)
    {
      const double4 gq = pr.grid[best_g];
      const Qd q{gq.x, gq.y, gq.z, gq.w};
      for (uint32_t a = lane; a < n; a += 32) st3(P, a, rotated_about(ld3(P, a), c, q));
    }
    __syncwarp();
    double score = best_s;
    if (lane == 0) {
      b.rs_align_index[item] = best_g;
      b.rs_align_score[item] = best_s;
    }
    // (the final pose and dihedrals are replayed by K2 from the decision trace)

    // ---- dihedral sweep: num_repetitions x optimize_pass (docking.cpp:155-167, 197-215)
    bool failed = false;
    for (uint32_t rep = 0; rep < pr.reps && !failed; ++rep) {
      for (uint32_t r = 0; r < R && !failed; ++r) {
        const uint2 ij = b.rots[m.rot_base + r];
        const uint32_t* mm = b.masks + m.mask_base + r * W;
        const V3d pi = ld3(P, ij.x);
        const V3d delta = vsub(ld3(P, ij.y), pi);
        const double len = __dsqrt_rn(vdot(delta, delta));
        const V3d axis = vscale(__ddiv_rn(1.0, len), delta);
        bool committed = false;
        uint32_t bk = 0;
        double bs = 0.0;
        // dihedral_step (docking.cpp:127-149): every candidate scored and bump-checked.
        for (uint32_t k = 0; k < pr.S; ++k) {
          const double* X = P;
          if (k > 0) {
            if (len < 1e-12) {  // rotate_fragment's DegenerateAxisError (molecule.cpp:156-158)
              if (lane == 0) raise_error(b, GD_ERR_DEGENERATE_AXIS, lig);
              failed = true;
              break;
            }
            const double4 dt = pr.dtab[k];
            const Qd q{dt.x, __dmul_rn(axis.x, dt.y), __dmul_rn(axis.y, dt.y), __dmul_rn(axis.z, dt.y)};
            for (uint32_t a = lane; a < n; a += 32) {
              const bool mv = ((__ldg(mm + (a >> 5)) >> (a & 31)) & 1u) && a != ij.y;
              st3(Cd, a, mv ? rotated_about(ld3(P, a), pi, q) : ld3(P, a));
            }
            __syncwarp();
            X = Cd;
          }
          // score_pose (scoring.cpp:40-45): samples in parallel, index-order sum on lane 0.
          for (uint32_t a = lane; a < n; a += 32) S[a] = sample_exact(pk, ld3(X, a));
          __syncwarp();
          double s = 0.0;
          if (lane == 0) {
            double sum = 0.0;
            for (uint32_t a = 0; a < n; ++a) sum = __dadd_rn(sum, S[a]);
            s = __ddiv_rn(sum, double(n));
          }
          s = __shfl_sync(0xffffffffu, s, 0);
          // bump_check (scoring.cpp:47-61): all non-bonded pairs, equality passes.
          bool clash = false;
          for (uint32_t a = 0; a + 1 < n && !clash; ++a) {
            const V3d pa = ld3(X, a);
            const double ra = b.atoms[m.atom_base + a].w;
            const uint32_t* row = b.adj + m.adj_base + a * W;
            bool mine = false;
            for (uint32_t bb = a + 1 + lane; bb < n; bb += 32) {
              if (bit_of(row, bb)) continue;
              mine |= pair_clash_exact(pa, ld3(X, bb), ra, b.atoms[m.atom_base + bb].w, pr.clash);
            }
            clash = __any_sync(0xffffffffu, mine);
          }
          if (!clash && (!committed || s > bs)) {
            committed = true;
            bk = k;
            bs = s;
          }
          __syncwarp();
        }
        if (failed) break;
        if (committed) {
          if (bk != 0) {  // commit = rotate_fragment(current, r, k*delta) recomputed bit-exactly
            const double4 dt = pr.dtab[bk];
            const Qd q{dt.x, __dmul_rn(axis.x, dt.y), __dmul_rn(axis.y, dt.y), __dmul_rn(axis.z, dt.y)};
            for (uint32_t a = lane; a < n; a += 32) {
              const bool mv = ((__ldg(mm + (a >> 5)) >> (a & 31)) & 1u) && a != ij.y;
              if (mv) st3(P, a, rotated_about(ld3(P, a), pi, q));
            }
          }
          score = bs;
        }
        if (lane == 0) {
          b.rs_step_k[size_t(m.rot_base) * N * pr.reps + (size_t(rs) * pr.reps + rep) * R + r] =
              committed ? int32_t(bk) : -1;
        }
        __syncwarp();
      }
    }
    if (failed) break;
    // ---- restart result
    if (lane == 0) b.rs_score[item] = score;
    if (lane == 0) atomicAdd(b.stats + (list_mode ? 7 : 0), 1ull);
    __syncwarp();
  }
}

// --------------------------------------------------------------------------------------------
// K2: best restart per ligand (finish_dock, docking.cpp:208-225), then its final pose and
// dihedrals REPLAYED in FP64 from the decision trace instead of stored per restart: start pose
// (docking.cpp:52-69) -> the chosen grid rotation (apply_rotation_choice, :110-118) -> every
// committed k != 0 in order (rotate_fragment, molecule.cpp:145-174). The operations are K1's, in
// K1's order, so the bits are K1's; no per-restart pose or dihedral scratch exists. Warp per
// ligand, the pose in the warp's shared slot (3 max_n doubles).
// --------------------------------------------------------------------------------------------
__global__ void finalize_kernel(DevParams pr, DevBatch b) {
  extern __shared__ double k2_smem[];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lig = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (lig >= b.n_lig) return;
  // after a device-side error (DegenerateAxisError, ...) the K1 kernels stop early and the batch's
  // results are discarded: the trace may be incomplete, so there is nothing to replay
  if (*(volatile int*)b.error != 0) return;
  double* P = k2_smem + size_t(threadIdx.x >> 5) * 3 * b.max_n;
  const uint32_t N = pr.n_restarts;
  const LigMeta m = b.meta[lig];
  const uint32_t n = m.n, R = m.nr, W = (n + 31) / 32;
  double best = 0.0;
  uint32_t id = 0;
  for (uint32_t p = 0; p < N; ++p) {  // strict >: lowest restart id on ties
    const double s = b.rs_score[size_t(lig) * N + p];
    if (p == 0 || s > best) {
      best = s;
      id = p;
    }
  }
  if (lane == 0) {
    b.best_score[lig] = best;
    b.best_restart[lig] = id;
  }
  if (N == 0) {  // no restart: no pose (the flat outputs are zeros; the adapter returns empty)
    for (uint32_t a = lane; a < 3u * n; a += 32) b.final_xyz[size_t(m.atom_base) * 3 + a] = 0.0;
    for (uint32_t r = lane; r < R; r += 32) b.final_dih[m.rot_base + r] = 0.0;
    return;
  }
  const size_t item = size_t(lig) * N + id;
  for (uint32_t a = lane; a < n; a += 32) {
    const double4 at = b.atoms[m.atom_base + a];
    st3(P, a, V3d{at.x, at.y, at.z});
  }
  __syncwarp();
  {  // generate_starting_pose (docking.cpp:52-69)
    const V3d c0 = centroid_smem(P, n);
    const double4 q4 = b.start[2 * item], t4 = b.start[2 * item + 1];
    const Qd qs{q4.x, q4.y, q4.z, q4.w};
    const V3d tgt{t4.x, t4.y, t4.z};
    __syncwarp();
    for (uint32_t a = lane; a < n; a += 32) st3(P, a, vadd(qapply(qs, vsub(ld3(P, a), c0)), tgt));
    __syncwarp();
  }
  {  // apply_rotation_choice (docking.cpp:110-118) of the restart's alignment decision
    const V3d cen = centroid_smem(P, n);
    const double4 gq = pr.grid[b.rs_align_index[item]];
    const Qd q{gq.x, gq.y, gq.z, gq.w};
    __syncwarp();
    for (uint32_t a = lane; a < n; a += 32) st3(P, a, rotated_about(ld3(P, a), cen, q));
    __syncwarp();
  }
  for (uint32_t r = lane; r < R; r += 32) b.final_dih[m.rot_base + r] = b.dih0[m.rot_base + r];
  __syncwarp();
  const int32_t* trace = b.rs_step_k + size_t(m.rot_base) * N * pr.reps + size_t(id) * pr.reps * R;
  for (uint32_t st = 0; st < pr.reps * R; ++st) {
    const int32_t k = trace[st];
    if (k <= 0) continue;
    const uint32_t r = st % R;
    const uint2 ij = b.rots[m.rot_base + r];
    const uint32_t* mm = b.masks + m.mask_base + r * W;
    const V3d pi = ld3(P, ij.x);
    const V3d delta = vsub(ld3(P, ij.y), pi);
    const V3d axis = vscale(__ddiv_rn(1.0, __dsqrt_rn(vdot(delta, delta))), delta);
    const double4 dt = pr.dtab[k];
    const Qd q{dt.x, __dmul_rn(axis.x, dt.y), __dmul_rn(axis.y, dt.y), __dmul_rn(axis.z, dt.y)};
    __syncwarp();
    for (uint32_t a = lane; a < n; a += 32) {
      const bool mv = ((__ldg(mm + (a >> 5)) >> (a & 31)) & 1u) && a != ij.y;
      if (mv) st3(P, a, rotated_about(ld3(P, a), pi, q));
    }
    if (lane == 0) {  // molecule.cpp:170-172
      double d = fmod(__dadd_rn(b.final_dih[m.rot_base + r], dt.z), 2.0 * 3.14159265358979323846);
      if (d < 0.0) d = __dadd_rn(d, 2.0 * 3.14159265358979323846);
      b.final_dih[m.rot_base + r] = d;
    }
    __syncwarp();
  }
  double* dst = b.final_xyz + size_t(m.atom_base) * 3;
  for (uint32_t a = lane; a < 3u * n; a += 32) dst[a] = P[a];
}

__global__ void order_keys_kernel(DevPocket pk, DevBatch b, uint32_t n_items, uint32_t* keys, uint32_t* vals);

cudaError_t launch_dock(const DevPocket& pk, const DevParams& pr, const DevBatch& b_in, int n_sms,
                        cudaStream_t stream, int* launches, cudaEvent_t* ev, cudaStream_t stream_b,
                        cudaEvent_t mid) {
  // Morton item order only where K1a reads the cells through L1 (with the cells in shared memory
  // the natural order is as fast and skips the sort: C2 -0.3 % / -1.1 % at clash 0.75 / 0.1)
  DevBatch b = b_in;
  if (b.order && k1a_cells_in_smem(pk, b.max_n)) b.order = nullptr;
  const bool split = stream_b && mid && stream_b != stream;
  *launches = 0;
  cudaError_t e = cudaMemsetAsync(b.work_counter, 0, 20 * sizeof(unsigned int), stream);
  if (e != cudaSuccess) return e;
  if (ev && (e = cudaEventRecord(ev[0], stream)) != cudaSuccess) return e;
  const uint32_t n_items = b.n_lig * pr.n_restarts;
  if (b.order && n_items > 0 && (pr.mode & 0xff) != GD_MODE_EXACT) {
    uint32_t* keys_in = b.order_scratch;
    uint32_t* keys_out = keys_in + n_items;
    uint32_t* vals_in = keys_out + n_items;
    order_keys_kernel<<<(n_items + 255) / 256, 256, 0, stream>>>(pk, b, n_items, keys_in, vals_in);
    ++*launches;
    size_t tb = b.order_tmp_bytes;
    e = cub::DeviceRadixSort::SortPairs(b.order_tmp, tb, keys_in, keys_out, vals_in, b.order, int(n_items), 0, 15,
                                        stream);
    if (e != cudaSuccess) return e;
  }
  // the FP64 kernel over the ligands with n >= min_n, on counter `ctr`
  auto launch_exact = [&](cudaStream_t st, uint32_t min_n, unsigned int* ctr, uint32_t list_mode = 0u) -> cudaError_t {
    const uint32_t stride = 7 * b.max_n;  // doubles per warp
    const size_t per_warp = size_t(stride) * sizeof(double);
    int warps = int((200 * 1024) / per_warp);
    if (warps > 32) warps = 32;
    if (warps < 1) warps = 1;
    const size_t smem = per_warp * warps;
    cudaError_t r = cudaFuncSetAttribute(dock_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (r != cudaSuccess) return r;
    DevBatch bx = b;
    bx.work_counter = ctr;
    dock_exact_kernel<<<n_sms, 32 * warps, smem, st>>>(pk, pr, bx, stride, min_n, list_mode);
    ++*launches;
    return cudaGetLastError();
  };
  if (b.n_lig > 0) {
    const int mode = pr.mode & 0xff;
    if (mode == GD_MODE_EXACT) {  // everything in FP64 (the reference's arithmetic throughout)
      if ((e = launch_exact(stream, 0u, b.work_counter)) != cudaSuccess) return e;
      if (ev && (e = cudaEventRecord(ev[1], stream)) != cudaSuccess) return e;
      if (split) {
        if ((e = cudaEventRecord(mid, stream)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(stream_b, mid, 0)) != cudaSuccess) return e;
      }
    } else {
      // the fast kernels for every ligand up to kFastMaxAtoms, one K1a + K1b pair per size class
      // present (n <= 32, <= 64, <= 128: NS = 1, 2, 4 from that class's ligands only, so a few
      // larger ligands do not put a whole batch on the NS = 4 kernels); a mixed batch's ligands
      // beyond 128 atoms get K1a (NS = 8) and then the FP64 kernel on their own counters
      int n_cls = 0;
      for (int c = 0; c < 3; ++c) n_cls += b.class_max_n[c] ? 1 : 0;
      for (int c = 0, k = 0; c < 3; ++c) {
        if (!b.class_max_n[c]) continue;
        DevBatch bf = b;
        bf.max_n = b.class_max_n[c];
        bf.fast_min_n = n_cls == 1 ? 0u : (c == 0 ? 0u : (c == 1 ? 32u : 64u));
        if (n_cls > 1) bf.work_counter = b.work_counter + 4 * (c + 1);
        const bool last = ++k == n_cls;
        // timing (non-split): ev[1] after the last class's K1a is the K1a / K1b boundary
        e = launch_fast(pk, pr, bf, n_sms, stream, split ? mid : (ev && last ? ev[1] : nullptr),
                        split ? stream_b : nullptr);
        if (e != cudaSuccess) return e;
        *launches += 3;  // K1a, K1r, K1b
      }
      // the restarts the fast sweeps handed over (usually none: one short launch)
      if ((e = launch_exact(split ? stream_b : stream, 0u, b.work_counter + 18, 1u)) != cudaSuccess) return e;
      if (b.max_n > kFastMaxAtoms) {
        // ligands beyond 128 atoms: K1a (NS = 8) for their candidates, then the FP64 kernel
        DevBatch bb = b;
        bb.fast_min_n = kFastMaxAtoms;
        bb.work_counter = b.work_counter + 16;
        if ((e = launch_align_big(pk, pr, bb, n_sms, stream)) != cudaSuccess) return e;
        ++*launches;
        if (split) {
          if ((e = cudaEventRecord(mid, stream)) != cudaSuccess) return e;
          if ((e = cudaStreamWaitEvent(stream_b, mid, 0)) != cudaSuccess) return e;
        }
        if ((e = launch_exact(split ? stream_b : stream, kFastMaxAtoms + 1, b.work_counter + 2)) != cudaSuccess)
          return e;
      }
    }
    if (split) stream = stream_b;  // K2 follows K1b
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  } else if (ev && (e = cudaEventRecord(ev[1], stream)) != cudaSuccess) {
    return e;
  }
  if (ev && (e = cudaEventRecord(ev[2], stream)) != cudaSuccess) return e;
  if (b.n_lig > 0) {
    // up to 4 warps, one ligand each, 3 max_n doubles of pose per warp (within 200 KB)
    const size_t per_warp = 3 * size_t(b.max_n) * sizeof(double);
    const uint32_t warps = uint32_t(std::max<size_t>(1, std::min<size_t>(4, (200 * 1024) / per_warp)));
    const uint32_t threads = 32 * warps;
    const uint32_t blocks = (b.n_lig * 32 + threads - 1) / threads;
    const size_t smem = size_t(warps) * per_warp;
    if (smem > 48 * 1024 &&
        (e = cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) != cudaSuccess)
      return e;
    finalize_kernel<<<blocks, threads, smem, stream>>>(pr, b);
    ++*launches;
  }
  if (ev && (e = cudaEventRecord(ev[3], stream)) != cudaSuccess) return e;
  return cudaGetLastError();
}

// --------------------------------------------------------------------------------------------
// K3: top-k. Scores are non-negative doubles, so their bit patterns sort like the values; a
// stable descending radix sort keeps equal scores in ascending ligand order.
// --------------------------------------------------------------------------------------------
__global__ void topk_prepare(const double* score, uint32_t n, unsigned long long* keys, uint32_t* vals) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = __double_as_longlong(score[i]);
  vals[i] = i;
}

__global__ void topk_emit(const unsigned long long* keys, const uint32_t* vals, const uint32_t* restart,
                          uint32_t k, gd_hit* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  out[i].best_score = __longlong_as_double(keys[i]);
  out[i].ligand = vals[i];
  out[i].restart = restart[vals[i]];
}

// --------------------------------------------------------------------------------------------
// Item order: where K1a reads the cells through L1 (C5's 1.56 MB of cells do not fit shared
// memory), the fast kernels claim (ligand, restart) items sorted by the Morton code of the start
// target (32 buckets per axis of the pocket box). Work in flight at any moment then sits in a small
// region of the pocket, so the cells its samples gather stay in L1. Where the cells fit shared
// memory, launch_dock keeps ligand order (no sort).
// --------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 5 bits -> every third bit
  v &= 31u;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

__global__ void order_keys_kernel(DevPocket pk, DevBatch b, uint32_t n_items, uint32_t* keys, uint32_t* vals) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  const double4 t = b.start[2 * size_t(i) + 1];
  uint32_t c[3];
  const double tc[3] = {t.x, t.y, t.z};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double u = (tc[a] - pk.origin[a]) / (pk.spacing * double(pk.dims[a] - 1)) * 32.0;
    c[a] = u <= 0.0 ? 0u : (u >= 31.0 ? 31u : uint32_t(u));
  }
  keys[i] = spread3(c[0]) | (spread3(c[1]) << 1) | (spread3(c[2]) << 2);
  vals[i] = i;
}

size_t order_tmp_bytes(uint32_t n) {
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, int(n > 0 ? n : 1), 0, 15);
  return temp + 256;
}

size_t topk_scratch_bytes(uint32_t n) {
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, temp, (unsigned long long*)nullptr,
                                            (unsigned long long*)nullptr, (uint32_t*)nullptr,
                                            (uint32_t*)nullptr, int(n));
  return temp + 2 * n * (sizeof(unsigned long long) + sizeof(uint32_t)) + 256;
}

cudaError_t launch_topk(const DevBatch& b, uint32_t k, void* scratch, size_t bytes, gd_hit* out,
                        cudaStream_t stream) {
  const uint32_t n = b.n_lig;
  char* p = static_cast<char*>(scratch);
  auto* k_in = reinterpret_cast<unsigned long long*>(p);
  auto* k_out = k_in + n;
  auto* v_in = reinterpret_cast<uint32_t*>(k_out + n);
  auto* v_out = v_in + n;
  char* temp = reinterpret_cast<char*>(v_out + n);
  temp = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(temp) + 255) & ~uintptr_t(255));
  size_t temp_bytes = bytes - size_t(temp - p);
  topk_prepare<<<(n + 255) / 256, 256, 0, stream>>>(b.best_score, n, k_in, v_in);
  cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(temp, temp_bytes, k_in, k_out, v_in, v_out,
                                                            int(n), 0, 64, stream);
  if (e != cudaSuccess) return e;
  if (k > n) k = n;
  if (k) topk_emit<<<(k + 255) / 256, 256, 0, stream>>>(k_out, v_out, b.best_restart, k, out);
  return cudaGetLastError();
}

}  // namespace gdk
