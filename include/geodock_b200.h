/*
 * geodock_b200 — C-ABI of the B200-native GeoDock pose search (arXiv 1901.06229 hot path).
 *
 * Drop-in boundary for the reference's plugin entry points (paths relative to
 * /root/reference/proj):
 *
 *   DockResult dock_ligand(const Ligand&, const Pocket&, const DockParams&, DockStats*)
 *       include/geodock/docking.hpp:140-141, src/docking.cpp:237-244
 *   run_screening(library, pocket, params, NodeConfig, PipelineHooks) -> (results, RunMetrics)
 *       include/geodock/pipeline.hpp:85-89, src/pipeline.cpp:187-290
 *
 * Both become gd_dock_batch(): a batch of ligands in, one result per ligand out (library order),
 * each result bit-identical to dock_ligand on the same inputs. No exceptions cross this boundary:
 * every entry point returns a GD_* status and gd_last_error(ctx) holds the message the reference
 * would have thrown (errors.hpp:10-67). Plain pointers and sizes only; the caller owns every host
 * buffer, the context owns every device buffer. A context is bound to one GPU and is externally
 * synchronized (mirrors DeviceLane::guard, pipeline.cpp:75,138); different GPUs' contexts run
 * concurrently.
 */
#ifndef GEODOCK_B200_H
#define GEODOCK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. The C++ adapter rethrows the matching geodock:: exception. */
#define GD_OK 0
#define GD_ERR_ARGUMENT 1        /* bad pointer / size at the ABI itself                       */
#define GD_ERR_INVALID_LIGAND 2  /* ValidationError   (docking.cpp:239-240, molecule.cpp:176-238) */
#define GD_ERR_CONTRACT 3        /* ContractError     (geometry.cpp:18-20, scoring.cpp:41,48-50) */
#define GD_ERR_DEGENERATE_AXIS 4 /* DegenerateAxisError (molecule.cpp:156-158)                 */
#define GD_ERR_CUDA 5            /* device / runtime failure (no CPU fallback exists)           */
#define GD_ERR_NO_POCKET 6       /* gd_dock_* before gd_set_pocket                              */
#define GD_ERR_UNSUPPORTED 7     /* ligand larger than GD_MAX_ATOMS (the FP64 kernel's per-warp
                                    shared-memory pose, 7 doubles per atom in 200 KB)          */
#define GD_ERR_PARSE 8           /* ParseError        (errors.hpp:15-27): malformed .lgd text     */

#define GD_MAX_ATOMS 3584         /* per ligand (the reference has no fixed limit): <= 128 atoms
                                    run the two-stage fast kernels, 129..256 the coarse K1a screen
                                    + the FP64 sweep, larger ones the all-FP64 kernel             */
#define GD_MAX_ROTAMERS 128       /* kMaxRotamers, molecule.hpp:29                              */

typedef struct gd_ctx gd_ctx;
typedef struct gd_batch gd_batch;
typedef struct gd_libbuf gd_libbuf;
typedef struct gd_pocketbuf gd_pocketbuf;

/* DockParams (docking.hpp:15-22). gd_default_params() returns the reference defaults. */
typedef struct {
  uint32_t n_restarts;        /* 32 */
  uint32_t num_repetitions;   /* 3 */
  uint32_t rotation_steps[3]; /* {16,16,8} */
  uint32_t dihedral_steps;    /* 36 */
  double clash_factor;        /* 0.75 */
  uint64_t seed;              /* 0 */
} gd_params;

/* A ligand library in flat SoA form (Ligand/Atom/Rotamer, molecule.hpp:12-46). Ligand l owns
 * atoms [atom_off[l], atom_off[l+1]), bonds [bond_off[l], bond_off[l+1]) and rotamers
 * [rot_off[l], rot_off[l+1]); bond and rotamer atom indices are local to the ligand.
 * dihedrals may be NULL (all zero, as make_ligand leaves them). Names are not NUL-terminated:
 * ligand l's name is names[name_off[l] .. name_off[l+1]). */
typedef struct {
  uint32_t n_ligands;
  const uint32_t* atom_off;  /* [n_ligands+1] */
  const double* xyz;         /* [3*atoms]     */
  const double* radius;      /* [atoms]       */
  const uint32_t* bond_off;  /* [n_ligands+1] */
  const uint32_t* bonds;     /* [2*bonds]     */
  const uint32_t* rot_off;   /* [n_ligands+1] */
  const uint32_t* rots;      /* [2*rotamers] (atom_i, atom_j) */
  const double* dihedrals;   /* [rotamers] or NULL */
  const uint32_t* name_off;  /* [n_ligands+1] */
  const char* names;
} gd_library;

/* DockResult (docking.hpp:34-42), flat. Required: best_score, best_restart. Optional (NULL =
 * skip): score_calls, phase_times ([2*n]: align, optimize nominal seconds), final_xyz
 * ([3*atoms], atom-indexed like the input), final_dihedrals ([rotamers]).
 * Optional decision trace (for parity checks), with N = n_restarts, p = l*N + restart:
 *   align_index[p], align_score[p], restart_score[p],
 *   step_k[rot_off[l]*N*reps + (restart*reps + rep)*R_l + r]  (committed k, or -1). */
typedef struct {
  double* best_score;
  uint32_t* best_restart;
  uint64_t* score_calls;
  double* phase_times;
  double* final_xyz;
  double* final_dihedrals;
  uint32_t* align_index;
  double* align_score;
  double* restart_score;
  int32_t* step_k;
} gd_results;

/* One top-k record: ordered by best_score desc, then ligand index asc. */
typedef struct {
  double best_score;
  uint32_t ligand;      /* index within the staged batch (+ the caller's global offset) */
  uint32_t restart;
} gd_hit;

/* Kernel-side counters for the last gd_run (mirrors DockStats, docking.hpp:46-55, plus the
 * coarse/exact split of the two-stage search). */
typedef struct {
  uint64_t restarts;           /* (ligand, restart) work items processed            */
  uint64_t align_exact_evals;  /* FP64 re-scored alignment candidates              */
  uint64_t align_fallbacks;    /* restarts whose alignment fell back to full FP64   */
  uint64_t step_exact_evals;   /* FP64 re-scored dihedral candidates               */
  uint64_t step_fallbacks;     /* restarts the fast sweep handed to the FP64 kernel (razor-thin
                                  pairs in a moving fragment, non-tree layouts, S outside [2,64]) */
  uint64_t commits;            /* committed dihedral steps                          */
  uint64_t h2d_bytes;          /* bytes uploaded by the last gd_stage               */
  uint64_t d2h_bytes;          /* bytes downloaded by the last gd_fetch             */
  uint32_t launches;           /* kernels launched by the last gd_run               */
  uint32_t exact_fallback;     /* 1: the pocket field lies outside [0,1] (outside the
                                  Pocket contract, scoring.hpp:15), so the batch ran the
                                  all-FP64 kernel instead of the two-stage fast path   */
  uint64_t align_second_passes; /* restarts whose candidates K1a collected in a second
                                   coarse pass (a lane's top-4 overflowed)              */
  /* executed dihedral-sweep work of the fast kernel (the roofline numerator) */
  uint64_t sweep_steps;           /* dihedral steps (restart x rep x rotamer)              */
  uint64_t sweep_invariant_steps; /* steps with an invariant clash (no candidate eligible) */
  uint64_t sweep_scored_steps;    /* steps whose S-1 candidates were scored                */
  uint64_t sweep_samples;         /* moved-atom samples of the scored candidates           */
  uint64_t cross_pairs;           /* bump cross pairs (moved x fixed x candidate) evaluated */
  uint64_t sweep_moves;           /* k != 0 commits (the pose changed: its caches are refreshed) */
  uint64_t step_exact_score_evals;  /* FP64 candidate scores: near the best coarse score     */
  uint64_t step_exact_allout_evals; /* FP64 candidate scores: every moved atom outside (one per step) */
  uint64_t step_exact_face_evals;   /* FP64 candidate scores: a moved atom within ptol of a face */
  uint64_t step_exact_clash_evals;  /* FP64 cross-pair checks of candidates near the bump threshold */
} gd_stats;

/* Kernel variants. FAST = two-stage (FP32 coarse screen + exact FP64 refinement, bit-identical
 * decisions); EXACT = every score and bump test in FP64 (reference arithmetic, slow, the
 * fallback the fast path proves itself against). SKIP_INVARIANT_CLASH (FAST only) skips scoring
 * dihedral steps whose invariant pairs already clash (identical decisions; reported separately). */
#define GD_MODE_FAST 0
#define GD_MODE_EXACT 1
#define GD_FLAG_SKIP_INVARIANT_CLASH 0x100

gd_params gd_default_params(void);

/* Number of visible CUDA devices (-1 if the runtime cannot be queried). */
int gd_device_count(void);
int gd_create(int device, gd_ctx** out);
void gd_destroy(gd_ctx* ctx);
const char* gd_last_error(const gd_ctx* ctx);
const char* gd_version(void);

/* Pocket (scoring.hpp:18-37): x-fastest FP64 field, dims >= 2 each. Uploaded once, immutable. */
int gd_set_pocket(gd_ctx* ctx, const uint32_t dims[3], const double origin[3], double spacing,
                  const double* field);
/* Uploads the rotation grid (geometry.cpp:16-34) and the dihedral (cos, sin) table. */
int gd_set_params(gd_ctx* ctx, const gd_params* params);
int gd_set_mode(gd_ctx* ctx, int mode_and_flags);

/* dock_ligand / run_screening for a whole batch: validate + pack on the host, H2D, kernels, D2H,
 * pipelined over chunks of the library (host packing of chunk c+1 overlaps the GPU work of chunk
 * c; pinned staging and device arenas are kept by the context between calls). Synchronous.
 * Results are written in library order. */
int gd_dock_batch(gd_ctx* ctx, const gd_library* lib, gd_results* out);

/* Split form used by the benchmark: stage (validate + pack + H2D, resident), run (kernels only,
 * enqueued on the context stream, no host sync), fetch (D2H + unpack, synchronous). */
int gd_stage(gd_ctx* ctx, const gd_library* lib, gd_batch** out);
int gd_run(gd_batch* batch);
int gd_fetch(gd_batch* batch, gd_results* out);
int gd_topk(gd_batch* batch, uint32_t k, gd_hit* out, uint32_t* n_out);
void gd_batch_free(gd_batch* batch);
int gd_sync(gd_ctx* ctx);
void* gd_stream(gd_ctx* ctx);           /* cudaStream_t of the context */
int gd_last_stats(gd_ctx* ctx, gd_stats* out);
/* Device time (ms) of the last gd_run's kernels: ms[0] K1a coarse alignment, ms[1] K1b exact
 * refinement + dihedral sweep, ms[2] K2 finalize (CUDA events on the context stream). */
int gd_last_kernel_ms(gd_ctx* ctx, float* ms, uint32_t n);
/* Device accounting of the last gd_dock_batch (seconds), the GPU fields of RunMetrics
 * (pipeline.hpp:43-72, replaces the lane busy/idle bookkeeping of pipeline.cpp:32-183):
 * out[0] busy span (first chunk's K1a start to last chunk's K2 end), out[1] alignment (K1a) and
 * out[2] optimisation (K1b + K2) as per-chunk event intervals (chunks overlap, so these may sum to
 * more than out[0]), out[3] host time spent waiting for the GPU. */
int gd_last_run_times(gd_ctx* ctx, double* out, uint32_t n);

/* Closed-form scoring-call count, count_score_calls (docking.cpp:44-50). */
uint64_t gd_count_score_calls(const gd_params* params, uint64_t n_rotamers);

/* Ligand checks (validate_ligand, molecule.cpp:176-238) without a GPU: returns the number of
 * violations of ligand l; their text ('\n'-separated) goes to msg (truncated to cap). */
int gd_validate_ligand(const gd_library* lib, uint32_t l, char* msg, uint32_t cap);
/* Moving set of rotamer r of ligand l (finalize_ligand, molecule.cpp:80-99), sorted. */
int gd_moving_set(const gd_library* lib, uint32_t l, uint32_t r, uint32_t* out, uint32_t* out_len);

/* Ligand ingest: parse_ligand_library (io.cpp:96-140) over a whole .lgd text (len bytes, not
 * NUL-terminated), multi-threaded on the host. Every record is validated like the reference's
 * parser does (validate_ligand after "end"); the first failure in stream order is reported with
 * the reference's message (ParseError text with its 1-based line, or ValidationError) into err.
 * On success *out owns the library; gd_libbuf_view points a gd_library at it (dihedrals zero,
 * io.cpp:134); gd_libbuf_free releases it. No GPU needed. */
int gd_parse_library(const char* text, size_t len, gd_libbuf** out, char* err, uint32_t cap);
int gd_libbuf_view(const gd_libbuf* buf, gd_library* view);
void gd_libbuf_free(gd_libbuf* buf);
/* parse_pocket (io.cpp:162-206): .pkt text -> dims, origin, spacing, x-fastest field (ParseError /
 * RangeError messages as the reference's). gd_pocketbuf_view's field pointer lives until free. */
int gd_parse_pocket(const char* text, size_t len, gd_pocketbuf** out, char* err, uint32_t cap);
int gd_pocketbuf_view(const gd_pocketbuf* buf, uint32_t dims[3], double origin[3], double* spacing,
                      const double** field);
void gd_pocketbuf_free(gd_pocketbuf* buf);

/* Host-side half of gd_stage without a GPU (diagnostics): validation + SoA packing of the whole
 * library into the device layout, on `threads` host threads (0: the context default, see
 * GD_HOST_THREADS). *seconds = wall time. Status as gd_stage's validation. */
int gd_host_pack(const gd_library* lib, const gd_params* params, const uint32_t dims[3], const double origin[3],
                 double spacing, uint32_t threads, double* seconds);

/* Synthetic inputs (generate.hpp:12-31), host-side and deterministic in the seed. */
int gd_make_pocket(const uint32_t dims[3], double spacing, const double origin[3], uint32_t blobs,
                   uint64_t seed, double* field_out);
/* Every generated ligand has `atoms` atoms, atoms-1 bonds, min(rotamers, atoms-1) rotamers;
 * outputs are sized accordingly (names are "lig_%06zu" and are not written here). */
int gd_make_library(uint64_t count, uint64_t atoms, uint64_t rotamers, uint64_t seed,
                    double* xyz, double* radius, uint32_t* bonds, uint32_t* rots);
/* Ligands [first, first + count) of the same library (each ligand has its own random stream,
 * generate.cpp:76), e.g. one rank's shard of a 1M-ligand screen; outputs sized for count ligands. */
int gd_make_library_range(uint64_t first, uint64_t count, uint64_t atoms, uint64_t rotamers, uint64_t seed,
                          double* xyz, double* radius, uint32_t* bonds, uint32_t* rots);

#ifdef __cplusplus
}
#endif
#endif /* GEODOCK_B200_H */
