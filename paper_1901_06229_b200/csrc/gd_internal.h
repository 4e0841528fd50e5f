// Internal layout shared by the host packer (gd_capi.cpp) and the kernels (gd_kernels.cu).
// Not part of the C-ABI. DESIGN.md §2 documents the HBM layout.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "geodock_b200.h"

namespace gdk {

constexpr uint32_t kFastMaxAtoms = 128;  // the fast kernels keep <= 128 atoms per warp in registers
constexpr uint32_t kAlignBigMaxAtoms = 256;  // K1a's coarse screen (NS = 8) for the FP64 sweep's ligands
constexpr int kAlignCand = 64;      // alignment candidates handed from K1a to K1b per restart

// Per-ligand metadata (32 B, one coalesced load per warp).
struct LigMeta {
  uint32_t atom_base;  // first atom in atoms[] / final_xyz
  uint32_t rot_base;   // first rotamer in rots[] / dih0[]
  uint32_t mask_base;  // moving bitmask of rotamer r: masks[mask_base + r*W .. +W)
  uint32_t adj_base;   // bonded row of atom a: adj[adj_base + a*W .. +W)
  uint16_t n;          // atoms
  uint16_t nr;         // rotamers
  uint32_t fast_ok;    // 1: every rotamer's moving set is a contiguous DFS range (fast sweep)
  uint32_t npad;       // atoms rounded up to a multiple of 4 (coarse alignment loop)
  uint32_t pad1;
};
static_assert(sizeof(LigMeta) == 32, "LigMeta layout");

// Pocket as seen by the kernels.
struct DevPocket {
  const double* field;   // FP64 x-fastest field (exact path)
  const uint4* cells;    // coarse cells (four quantised x-edges each, gd_set_pocket), (mx*my*mz)+1 entries
  uint32_t dims[3];
  uint32_t cell_dims[3]; // dims - 1
  double origin[3];
  double spacing;
  double inv_spacing;    // 1 / spacing (FP32 grid coordinates of the coarse path only)
  double maxc[3];        // dims - 1 as doubles (sample_field's outside test, scoring.cpp:16-18)
  float inv_spacing_f;
  float q_eps;           // quantisation bound of one coarse sample (inf: fast path off)
  float coarse_scale;    // scale of the decoded coarse values (1 with the current encoding)
  float dz_bias;         // B: bias of the cells' dD field (3, or 6 for second differences beyond 1)
  float max_step;        // max |v(i+1) - v(i)| along any axis: slope bound per grid unit
  const float* field_f;  // FP32 copy of the field (K1b's coarse samples) + a zero tail of f_tail floats
  uint32_t f_dummy, f_count;  // first float of the zero tail (samples outside the grid), total floats
  float q_eps_f;         // max |float(v) - v| over the field (K1b's quantisation term)
};

// Search parameters as seen by the kernels.
struct DevParams {
  const double4* grid;     // G rotation quaternions (w,x,y,z), FP64, host-built with libm
  const float4* grid_f;    // G x 3 float4 rows of R/spacing (coarse path)
  const double4* dtab;     // S entries: (cos(k*delta/2), sin(k*delta/2), k*delta, 0)
  const float2* dtab_f;    // S entries: (cos, sin) in FP32 (coarse path)
  const float4* frames;    // b*c x 3 float4 rows of Ry(beta_j) Rz(gamma_k) / spacing (separable coarse path)
  const uint32_t* frame_tab;  // twin lists + K1a work units of the separable coarse path (upload_grid_f)
  uint32_t n_kept;         // K1a work units (kept frame | c0 << 16); twin frames are not screened
  uint32_t n_twin_frames;  // frames folded into a kept frame (0: every frame is screened)
  float2 acs[16];          // (cos alpha_i, sin alpha_i), i < steps[0] (kernel parameter: constant bank)
  uint32_t steps[3];       // rotation_steps
  uint32_t n_restarts;
  uint32_t reps;
  uint32_t G;
  uint32_t S;
  double clash;
  float clash_f;
  int mode;                // GD_MODE_* | flags
};

// Device-resident batch.
struct DevBatch {
  uint32_t n_lig;
  uint32_t lig_base;       // library index of this batch's ligand 0 (executor chunks; error reports)
  uint32_t n_atoms;
  uint32_t n_rots;
  uint32_t max_n;
  uint32_t fast_max_n;     // largest n <= kFastMaxAtoms (the fast kernels' ligands; 0: none)
  uint32_t fast_min_n;     // the fast kernels of one launch take kFastClass-ligands with n > this
  uint32_t class_max_n[3]; // largest n per fast class (n <= 32, <= 64, <= 128; 0: class absent)
  const LigMeta* meta;
  const double4* atoms;    // (x, y, z, radius)
  const double4* start;    // per (ligand, restart): [q(w,x,y,z)], [t(x,y,z), 0]  -> 2 x double4
  const uint2* rots;       // (atom_i, atom_j)
  const double* dih0;      // initial dihedrals
  const uint32_t* masks;   // moving bitmasks
  const uint32_t* adj;     // bonded bitmask rows (original atom order)
  // fast-path layout: atoms in DFS preorder so every moving set is a contiguous range
  const uint16_t* dfs_pos; // original atom -> DFS position
  const ushort4* rdfs;     // per rotamer: (s = DFS pos of j, e = end of moving range, DFS pos of i, 0)
  const uint32_t* adjd;    // bonded bitmask rows in DFS space: adjd[adj_base + pos*W + w]
  // per-restart scratch / trace
  uint16_t* rs_cand;       // K1a -> K1b: alignment candidates of restart `item`, [item*kAlignCand ..)
  int32_t* rs_ncand;       // candidate count, or -1: full FP64 alignment (overflow / plateau)
  double* rs_score;
  double* rs_align_score;
  uint32_t* rs_align_index;
  int32_t* rs_step_k;      // rot_base*N*reps + (restart*reps + rep)*R + r
  // K1r -> K1b (fast path): the aligned FP64 pose of restart rs of ligand l at
  // rs_pose[3 (atom_base(l) N + rs n(l) + a) ..], its exact per-atom samples in rs_es (same index /
  // 3), and the ligand's extent about its centroid (the coarse position bound) in rs_ext[item]
  double* rs_pose;
  double* rs_es;
  float* rs_ext;
  // restarts K1b hands to the FP64 kernel (a step it cannot decide with its cached pair state:
  // razor-thin pairs inside the moving fragment, non-tree layouts, S outside [2, 64]); count in
  // work_counter[19]
  uint32_t* slow_items;
  unsigned int* slow_count;  // = the batch's work_counter + 19 (class launches keep this pointer)
  // per-ligand results
  double* best_score;
  uint32_t* best_restart;
  double* final_xyz;
  double* final_dih;
  // claim order of the fast kernels' items (sorted by start target, see launch_dock; nullptr:
  // natural order) and its sort scratch: keys in / keys out / values in (3 x n_items u32) + cub temp
  uint32_t* order;
  uint32_t* order_scratch;
  void* order_tmp;
  size_t order_tmp_bytes;
  // control
  unsigned int* work_counter;  // [0] K1 / K1b items, [1] K1a items
  int* error;              // [0] = status, [1] = ligand index
  unsigned long long* stats;  // gd_stats counters (6 x u64)
};

// Kernel launchers (gd_kernels.cu). Return cudaGetLastError() of the launches.
// ev (nullable): 4 events recorded around K1a, K1b and K2 (per-kernel timing).
// Pipelined form (stream_b and mid non-null): K1a on `stream`, then K1b and K2 on stream_b after
// `mid` — the executor keeps the alignment of chunk c+1 and the sweep of chunk c in flight together.
// cub temp bytes of the item-order sort for n items
size_t order_tmp_bytes(uint32_t n);
// quarter-turn groups of one K1a work unit (the unit table's c0 step, upload_grid_f; gd_fast.cu)
uint32_t k1a_qt_groups();
// K1a holds the pocket's cells in shared memory for ligands of up to max_n atoms (gd_fast.cu)
bool k1a_cells_in_smem(const DevPocket& pk, uint32_t max_n);

cudaError_t launch_dock(const DevPocket& pk, const DevParams& pr, const DevBatch& b, int n_sms,
                        cudaStream_t stream, int* launches, cudaEvent_t* ev = nullptr,
                        cudaStream_t stream_b = nullptr, cudaEvent_t mid = nullptr);
// Device top-k by (best_score desc, ligand asc) into out[0..k). Needs scratch from topk_scratch_bytes.
size_t topk_scratch_bytes(uint32_t n_lig);
cudaError_t launch_topk(const DevBatch& b, uint32_t k, void* scratch, size_t scratch_bytes,
                        gd_hit* out, cudaStream_t stream);

}  // namespace gdk
