// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" shim over the UNMODIFIED reference (GeoDock, /root/reference/proj), compiled
// together with the reference's own sources by oracle/Makefile into oracle/_ref/libgeodock_ref.so.
// Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference legs load it.
//
// Every entry point here calls the reference's public API; the shim only converts between the
// flat "library" layout used across this repo (include/geodock_b200.h, gd_library) and the
// reference's value types (Ligand/Pocket/DockParams, proj/include/geodock/*.hpp).
//
// The trace entry point (ref_dock_trace) re-runs the reference's own decomposed pieces in the same
// order dock_ligand uses them (docking.cpp:237-244 → align_restarts :178-195 → finish_dock
// :197-235, with optimize_pass :155-167 inlined because it is file-static) to expose the per-restart
// alignment choice and the per-(rep, rotamer) dihedral decisions, and asserts the composed result
// is bit-identical to dock_ligand's.

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "geodock/docking.hpp"
#include "geodock/errors.hpp"
#include "geodock/generate.hpp"
#include "geodock/io.hpp"
#include "geodock/molecule.hpp"
#include "geodock/pipeline.hpp"
#include "geodock/prng.hpp"
#include "geodock/scoring.hpp"
#include "testkit/testkit.hpp"

using namespace geodock;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

// Status codes shared with include/geodock_b200.h.
constexpr int kOk = 0;
constexpr int kInvalidLigand = 2;
constexpr int kContract = 3;
constexpr int kDegenerate = 4;
constexpr int kOther = 9;

Pocket make_pocket_from(const uint32_t dims[3], const double origin[3], double spacing,
                        const double* field) {
  Pocket p;
  p.origin = {origin[0], origin[1], origin[2]};
  p.spacing = spacing;
  p.dims = {dims[0], dims[1], dims[2]};
  const std::size_t n = std::size_t(dims[0]) * dims[1] * dims[2];
  p.field.assign(field, field + n);
  return p;
}

DockParams params_from(uint32_t n_restarts, uint32_t reps, const uint32_t steps[3],
                       uint32_t dihedral_steps, double clash, uint64_t seed) {
  DockParams p;
  p.n_restarts = n_restarts;
  p.num_repetitions = reps;
  p.rotation_steps = {steps[0], steps[1], steps[2]};
  p.dihedral_steps = dihedral_steps;
  p.clash_factor = clash;
  p.seed = seed;
  return p;
}

// Builds ligand `l` of a flat library through the reference's own constructor (validate +
// finalize, molecule.cpp:101-115), then overrides the dihedral state.
Ligand ligand_from(uint32_t l, const uint32_t* atom_off, const double* xyz, const double* radius,
                   const uint32_t* bond_off, const uint32_t* bonds, const uint32_t* rot_off,
                   const uint32_t* rots, const double* dihedrals, const uint32_t* name_off,
                   const char* names) {
  std::vector<Atom> atoms;
  for (uint32_t a = atom_off[l]; a < atom_off[l + 1]; ++a) {
    atoms.push_back({{xyz[3 * a], xyz[3 * a + 1], xyz[3 * a + 2]}, radius[a]});
  }
  std::vector<Bond> bl;
  for (uint32_t b = bond_off[l]; b < bond_off[l + 1]; ++b) bl.emplace_back(bonds[2 * b], bonds[2 * b + 1]);
  std::vector<Bond> rl;
  for (uint32_t r = rot_off[l]; r < rot_off[l + 1]; ++r) rl.emplace_back(rots[2 * r], rots[2 * r + 1]);
  std::string name(names + name_off[l], names + name_off[l + 1]);
  Ligand lig = make_ligand(std::move(name), std::move(atoms), std::move(bl), std::move(rl));
  if (dihedrals) {
    for (uint32_t r = rot_off[l]; r < rot_off[l + 1]; ++r) lig.dihedrals[r - rot_off[l]] = dihedrals[r];
  }
  return lig;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// make_pocket (generate.cpp:27-66). field_out has dims[0]*dims[1]*dims[2] doubles.
int ref_make_pocket(const uint32_t dims[3], double spacing, const double origin[3], uint32_t blobs,
                    uint64_t seed, double* field_out) {
  try {
    PocketSpec spec;
    spec.dims = {dims[0], dims[1], dims[2]};
    spec.spacing = spacing;
    spec.origin = {origin[0], origin[1], origin[2]};
    spec.blobs = blobs;
    spec.seed = seed;
    const Pocket p = make_pocket(spec);
    std::memcpy(field_out, p.field.data(), p.field.size() * sizeof(double));
    return kOk;
  } catch (const std::exception& e) {
    return fail(e, kOther);
  }
}

// make_library (generate.cpp:68-109), flattened. Every generated ligand has `atoms` atoms,
// atoms-1 bonds and min(rotamers, atoms-1) rotamers, so the caller sizes the outputs from those.
int ref_make_library(uint64_t count, uint64_t atoms, uint64_t rotamers, uint64_t seed, double* xyz,
                     double* radius, uint32_t* bonds, uint32_t* rots) {
  try {
    LibrarySpec spec;
    spec.count = count;
    spec.atoms = atoms;
    spec.rotamers = rotamers;
    spec.seed = seed;
    const std::vector<Ligand> lib = make_library(spec);
    std::size_t a = 0, b = 0, r = 0;
    for (const Ligand& lig : lib) {
      for (const Atom& at : lig.atoms) {
        xyz[3 * a] = at.position.x;
        xyz[3 * a + 1] = at.position.y;
        xyz[3 * a + 2] = at.position.z;
        radius[a] = at.radius;
        ++a;
      }
      for (const Bond& bd : lig.bonds) {
        bonds[2 * b] = uint32_t(bd.first);
        bonds[2 * b + 1] = uint32_t(bd.second);
        ++b;
      }
      for (const Rotamer& ro : lig.rotamers) {
        rots[2 * r] = uint32_t(ro.atom_i);
        rots[2 * r + 1] = uint32_t(ro.atom_j);
        ++r;
      }
    }
    return kOk;
  } catch (const std::exception& e) {
    return fail(e, kOther);
  }
}

// testkit::random_ligand / random_pocket specs (testkit.cpp:236-256) driven by a caller-held
// SplitMix64 state, so tests can reproduce acceptance #2 (acceptance_main.cpp:100-165).
// Returns the LibrarySpec / PocketSpec the testkit would build; the caller then calls
// ref_make_library / ref_make_pocket with them.
int ref_random_ligand_spec(uint64_t* rng_state, uint64_t max_atoms, uint64_t max_rotamers,
                           uint64_t* atoms, uint64_t* rotamers, uint64_t* seed) {
  SplitMix64 rng(*rng_state);
  const std::size_t n = 1 + rng.below(max_atoms);
  const std::size_t r = n > 1 ? rng.below(std::min<std::size_t>(max_rotamers, n - 1) + 1) : 0;
  *atoms = n;
  *rotamers = r;
  *seed = rng.next();
  *rng_state = rng.state;
  return kOk;
}

// Per-ligand minimum moving set of rotamer r as a sorted index list (molecule.cpp:80-99).
int ref_moving_set(uint32_t n_atoms, const double* xyz, const double* radius, uint32_t n_bonds,
                   const uint32_t* bonds, uint32_t n_rot, const uint32_t* rots, uint32_t r,
                   uint32_t* out, uint32_t* out_len) {
  try {
    uint32_t ao[2] = {0, n_atoms}, bo[2] = {0, n_bonds}, ro[2] = {0, n_rot}, no[2] = {0, 1};
    const Ligand lig = ligand_from(0, ao, xyz, radius, bo, bonds, ro, rots, nullptr, no, "x");
    const auto& ms = lig.rotamers.at(r).moving_set;
    for (std::size_t i = 0; i < ms.size(); ++i) out[i] = uint32_t(ms[i]);
    *out_len = uint32_t(ms.size());
    return kOk;
  } catch (const ValidationError& e) {
    return fail(e, kInvalidLigand);
  } catch (const std::exception& e) {
    return fail(e, kOther);
  }
}

// validate_ligand (molecule.cpp:176-238) on a raw (un-finalized) ligand: returns the number of
// violations and writes them '\n'-separated into msg (truncated to cap).
int ref_validate(uint32_t n_atoms, const double* xyz, const double* radius, uint32_t n_bonds,
                 const uint32_t* bonds, uint32_t n_rot, const uint32_t* rots, char* msg,
                 uint32_t cap) {
  Ligand lig;
  lig.name = "v";
  for (uint32_t a = 0; a < n_atoms; ++a) {
    lig.atoms.push_back({{xyz[3 * a], xyz[3 * a + 1], xyz[3 * a + 2]}, radius[a]});
  }
  for (uint32_t b = 0; b < n_bonds; ++b) lig.bonds.emplace_back(bonds[2 * b], bonds[2 * b + 1]);
  for (uint32_t r = 0; r < n_rot; ++r) lig.rotamers.push_back({rots[2 * r], rots[2 * r + 1], {}});
  lig.dihedrals.assign(n_rot, 0.0);
  const std::vector<std::string> v = validate_ligand(lig);
  std::string all;
  for (const auto& s : v) all += s + "\n";
  if (cap > 0) {
    std::snprintf(msg, cap, "%s", all.c_str());
  }
  return int(v.size());
}

// Rotation grid quaternions (geometry.cpp:16-34), [w,x,y,z] per entry.
int ref_rotation_grid(const uint32_t steps[3], double* q_out) {
  try {
    const RotationGrid g = enumerate_rotations(steps[0], steps[1], steps[2]);
    for (std::size_t i = 0; i < g.size(); ++i) {
      q_out[4 * i] = g[i].w;
      q_out[4 * i + 1] = g[i].x;
      q_out[4 * i + 2] = g[i].y;
      q_out[4 * i + 3] = g[i].z;
    }
    return kOk;
  } catch (const std::exception& e) {
    return fail(e, kContract);
  }
}

// sample_field (scoring.cpp:9-38) at n points.
int ref_sample_field(const uint32_t dims[3], const double origin[3], double spacing,
                     const double* field, uint64_t n, const double* pts, double* out) {
  const Pocket p = make_pocket_from(dims, origin, spacing, field);
  for (uint64_t i = 0; i < n; ++i) out[i] = sample_field(p, {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
  return kOk;
}

// mix_seed / fnv1a64 (prng.hpp:33-46).
uint64_t ref_fnv1a64(const char* s, uint64_t len) { return fnv1a64(std::string_view(s, len)); }
uint64_t ref_mix_seed(uint64_t a, uint64_t b) { return mix_seed(a, b); }

// Flat-library dock. Library layout = gd_library in include/geodock_b200.h.
// Outputs per ligand l: best_score[l], best_restart[l], score_calls[l], phase[2l..2l+1],
// final_xyz (atom-indexed like the input), final_dih (rotamer-indexed).
// Optional trace (any pointer may be null), per (ligand, restart) p = l*N + restart:
//   align_index[p], align_score[p], restart_score[p],
//   step_k[(rot_off[l]*N*reps) + (restart*reps + rep)*R_l + r]  (k, or -1 when nothing committed),
//   step_score[same index] (winning score when committed, else the carried score).
int ref_dock_library(uint32_t n_lig, const uint32_t* atom_off, const double* xyz,
                     const double* radius, const uint32_t* bond_off, const uint32_t* bonds,
                     const uint32_t* rot_off, const uint32_t* rots, const double* dihedrals,
                     const uint32_t* name_off, const char* names, const uint32_t dims[3],
                     const double origin[3], double spacing, const double* field,
                     uint32_t n_restarts, uint32_t reps, const uint32_t steps[3],
                     uint32_t dihedral_steps, double clash, uint64_t seed, double* best_score,
                     uint32_t* best_restart, uint64_t* score_calls, double* phase, double* final_xyz,
                     double* final_dih, uint32_t* align_index, double* align_score,
                     double* restart_score, int32_t* step_k, double* step_score) {
  uint32_t l = 0;
  try {
    const Pocket pocket = make_pocket_from(dims, origin, spacing, field);
    const DockParams params = params_from(n_restarts, reps, steps, dihedral_steps, clash, seed);
    const bool trace = align_index || align_score || restart_score || step_k || step_score;
    const RotationGrid grid = enumerate_rotations(params.rotation_steps);
    for (l = 0; l < n_lig; ++l) {
      const Ligand lig = ligand_from(l, atom_off, xyz, radius, bond_off, bonds, rot_off, rots,
                                     dihedrals, name_off, names);
      const DockResult res = dock_ligand(lig, pocket, params);
      best_score[l] = res.best_score;
      best_restart[l] = res.best_restart_id;
      score_calls[l] = res.score_calls;
      phase[2 * l] = res.phase_times.align_seconds;
      phase[2 * l + 1] = res.phase_times.optimize_seconds;
      for (std::size_t a = 0; a < res.final_coordinates.size(); ++a) {
        final_xyz[3 * (atom_off[l] + a)] = res.final_coordinates[a].x;
        final_xyz[3 * (atom_off[l] + a) + 1] = res.final_coordinates[a].y;
        final_xyz[3 * (atom_off[l] + a) + 2] = res.final_coordinates[a].z;
      }
      for (std::size_t r = 0; r < res.final_dihedrals.size(); ++r) final_dih[rot_off[l] + r] = res.final_dihedrals[r];
      if (!trace) continue;

      // Decomposed replay with the reference's public pieces (docking.cpp:178-235).
      const std::size_t R = lig.rotamers.size();
      double best = 0.0;
      bool have = false;
      unsigned best_id = 0;
      for (unsigned pid = 0; pid < params.n_restarts; ++pid) {
        const std::size_t p = std::size_t(l) * params.n_restarts + pid;
        const Ligand start = generate_starting_pose(lig, pid, params, pocket);
        const RotationChoice choice = best_rotation_in_range(start, pocket, grid, 0, grid.size());
        auto [pose, score] = apply_rotation_choice(start, grid, choice);
        if (align_index) align_index[p] = uint32_t(choice.index);
        if (align_score) align_score[p] = choice.score;
        for (unsigned rep = 0; rep < params.num_repetitions; ++rep) {
          for (std::size_t r = 0; r < R; ++r) {
            DihedralStep st = dihedral_step(pose, r, pocket, params.dihedral_steps,
                                            params.clash_factor);
            if (st.committed) {
              pose = std::move(st.pose);
              score = st.score;
            }
            const std::size_t si = std::size_t(rot_off[l]) * params.n_restarts * params.num_repetitions +
                                   (std::size_t(pid) * params.num_repetitions + rep) * R + r;
            if (step_k) step_k[si] = st.committed ? int32_t(st.k) : -1;
            if (step_score) step_score[si] = score;
          }
        }
        if (restart_score) restart_score[p] = score;
        if (!have || score > best) {
          have = true;
          best = score;
          best_id = pid;
        }
      }
      if (best != res.best_score || best_id != res.best_restart_id) {
        g_err = "decomposed replay disagrees with dock_ligand for ligand " + lig.name;
        return kOther;
      }
    }
    return kOk;
  } catch (const ValidationError& e) {
    g_err = std::string(e.what()) + " (ligand " + std::to_string(l) + ")";
    return kInvalidLigand;
  } catch (const DegenerateAxisError& e) {
    return fail(e, kDegenerate);
  } catch (const ContractError& e) {
    return fail(e, kContract);
  } catch (const std::exception& e) {
    return fail(e, kOther);
  }
}

// testkit::reference_dock (testkit.cpp:54-140) for one ligand of a flat library; used to pin that
// the reference's naive transcription equals dock_ligand on the instances the tests use.
int ref_reference_dock(uint32_t l, const uint32_t* atom_off, const double* xyz,
                       const double* radius, const uint32_t* bond_off, const uint32_t* bonds,
                       const uint32_t* rot_off, const uint32_t* rots, const uint32_t* name_off,
                       const char* names, const uint32_t dims[3], const double origin[3],
                       double spacing, const double* field, uint32_t n_restarts, uint32_t reps,
                       const uint32_t steps[3], uint32_t dihedral_steps, double clash,
                       uint64_t seed, double* best_score, uint32_t* best_restart) {
  try {
    const Pocket pocket = make_pocket_from(dims, origin, spacing, field);
    const DockParams params = params_from(n_restarts, reps, steps, dihedral_steps, clash, seed);
    const Ligand lig = ligand_from(l, atom_off, xyz, radius, bond_off, bonds, rot_off, rots,
                                   nullptr, name_off, names);
    const DockResult r = testkit::reference_dock(lig, pocket, params);
    *best_score = r.best_score;
    *best_restart = r.best_restart_id;
    return kOk;
  } catch (const std::exception& e) {
    return fail(e, kOther);
  }
}

// run_screening (pipeline.cpp:187-290) with n_workers CPU workers and no device lanes: the
// reference's production CPU path, timed by the caller. Writes best scores / restarts.
int ref_run_screening(uint32_t n_lig, const uint32_t* atom_off, const double* xyz,
                      const double* radius, const uint32_t* bond_off, const uint32_t* bonds,
                      const uint32_t* rot_off, const uint32_t* rots, const uint32_t* name_off,
                      const char* names, const uint32_t dims[3], const double origin[3],
                      double spacing, const double* field, uint32_t n_restarts, uint32_t reps,
                      const uint32_t steps[3], uint32_t dihedral_steps, double clash,
                      uint64_t seed, uint32_t n_workers, double* best_score,
                      uint32_t* best_restart, double* wall_seconds) {
  try {
    const Pocket pocket = make_pocket_from(dims, origin, spacing, field);
    const DockParams params = params_from(n_restarts, reps, steps, dihedral_steps, clash, seed);
    std::vector<Ligand> lib;
    lib.reserve(n_lig);
    for (uint32_t l = 0; l < n_lig; ++l) {
      lib.push_back(ligand_from(l, atom_off, xyz, radius, bond_off, bonds, rot_off, rots, nullptr,
                                name_off, names));
    }
    NodeConfig cfg;
    cfg.n_workers = n_workers;
    cfg.n_devices = 0;
    auto [results, metrics] = run_screening(lib, pocket, params, cfg);
    for (uint32_t l = 0; l < n_lig; ++l) {
      best_score[l] = results[l].best_score;
      best_restart[l] = results[l].best_restart_id;
    }
    *wall_seconds = metrics.wall_seconds;
    return kOk;
  } catch (const std::exception& e) {
    return fail(e, kOther);
  }
}

// parse_ligand_library (io.cpp:96-140) over a text, flattened like gd_library: the result stays
// in a thread-local holder; ref_parse_counts / ref_parse_fetch read it out. Returns 0, or the
// status of the exception (8 ParseError, 2 ValidationError, 9 other) with ref_last_error().
thread_local std::vector<Ligand> g_parsed;

int ref_parse_library(const char* text, uint64_t len) {
  g_parsed.clear();
  try {
    std::istringstream in(std::string(text, len));
    g_parsed = parse_ligand_library(in);
    return kOk;
  } catch (const ValidationError& e) {
    return fail(e, kInvalidLigand);
  } catch (const ParseError& e) {
    return fail(e, 8);
  } catch (const std::exception& e) {
    return fail(e, kOther);
  }
}

void ref_parse_counts(uint64_t* n_lig, uint64_t* n_atoms, uint64_t* n_bonds, uint64_t* n_rots, uint64_t* n_chars) {
  *n_lig = g_parsed.size();
  *n_atoms = *n_bonds = *n_rots = *n_chars = 0;
  for (const Ligand& l : g_parsed) {
    *n_atoms += l.atoms.size();
    *n_bonds += l.bonds.size();
    *n_rots += l.rotamers.size();
    *n_chars += l.name.size();
  }
}

void ref_parse_fetch(uint32_t* atom_off, double* xyz, double* radius, uint32_t* bond_off, uint32_t* bonds,
                     uint32_t* rot_off, uint32_t* rots, double* dihedrals, uint32_t* name_off, char* names) {
  uint32_t a = 0, b = 0, r = 0, c = 0;
  for (std::size_t l = 0; l < g_parsed.size(); ++l) {
    const Ligand& lig = g_parsed[l];
    atom_off[l] = a;
    bond_off[l] = b;
    rot_off[l] = r;
    name_off[l] = c;
    for (const Atom& at : lig.atoms) {
      xyz[3 * a] = at.position.x;
      xyz[3 * a + 1] = at.position.y;
      xyz[3 * a + 2] = at.position.z;
      radius[a++] = at.radius;
    }
    for (const Bond& bd : lig.bonds) {
      bonds[2 * b] = uint32_t(bd.first);
      bonds[2 * b + 1] = uint32_t(bd.second);
      ++b;
    }
    for (std::size_t q = 0; q < lig.rotamers.size(); ++q) {
      rots[2 * r] = uint32_t(lig.rotamers[q].atom_i);
      rots[2 * r + 1] = uint32_t(lig.rotamers[q].atom_j);
      dihedrals[r++] = lig.dihedrals[q];
    }
    for (char ch : lig.name) names[c++] = ch;
  }
  const std::size_t L = g_parsed.size();
  atom_off[L] = a;
  bond_off[L] = b;
  rot_off[L] = r;
  name_off[L] = c;
}

// serialize_ligand_library (io.cpp:143-160) of the last parsed library into out (cap bytes);
// returns the full length.
uint64_t ref_serialize_parsed(char* out, uint64_t cap) {
  std::ostringstream os;
  serialize_ligand_library(os, g_parsed);
  const std::string s = os.str();
  if (out && cap) std::memcpy(out, s.data(), std::min<uint64_t>(cap, s.size()));
  return s.size();
}

// write_results (io.cpp:216-223) of n flat DockResults into out (cap bytes); returns the length.
uint64_t ref_write_results(uint64_t n, const uint32_t* name_off, const char* names, const double* best_score,
                           const uint32_t* best_restart, const uint64_t* score_calls, const double* phase,
                           char* out, uint64_t cap) {
  std::vector<DockResult> rs(n);
  for (uint64_t l = 0; l < n; ++l) {
    rs[l].ligand_name.assign(names + name_off[l], names + name_off[l + 1]);
    rs[l].best_score = best_score[l];
    rs[l].best_restart_id = best_restart[l];
    rs[l].score_calls = score_calls[l];
    rs[l].phase_times.align_seconds = phase[2 * l];
    rs[l].phase_times.optimize_seconds = phase[2 * l + 1];
  }
  std::ostringstream os;
  write_results(os, rs);
  const std::string s = os.str();
  if (out && cap) std::memcpy(out, s.data(), std::min<uint64_t>(cap, s.size()));
  return s.size();
}

// write_metrics (io.cpp:225-245) of a RunMetrics / NodeConfig given as flat numbers; returns the
// length. busy/idle/wait: per-lane arrays of nb, ni, nw entries.
uint64_t ref_write_metrics(uint32_t n_workers, uint32_t n_devices, uint32_t lane_width, int synthetic,
                           uint64_t ligands, double wall, double throughput, const double* busy, uint32_t nb,
                           const double* idle, uint32_t ni, const double* wait, uint32_t nw, double align_total,
                           double optimize_total, uint64_t lane_failures, uint64_t violations, char* out,
                           uint64_t cap) {
  RunMetrics m;
  m.wall_seconds = wall;
  m.throughput = throughput;
  m.ligand_count = ligands;
  m.device_busy_seconds.assign(busy, busy + nb);
  m.device_idle_seconds.assign(idle, idle + ni);
  m.worker_wait_seconds.assign(wait, wait + nw);
  m.align_seconds_total = align_total;
  m.optimize_seconds_total = optimize_total;
  m.lane_failures = lane_failures;
  m.exclusivity_violations = violations;
  NodeConfig c;
  c.n_workers = n_workers;
  c.n_devices = n_devices;
  c.lane_width = lane_width;
  c.mode = synthetic ? ExecMode::synthetic : ExecMode::real;
  std::ostringstream os;
  write_metrics(os, m, c);
  const std::string s = os.str();
  if (out && cap) std::memcpy(out, s.data(), std::min<uint64_t>(cap, s.size()));
  return s.size();
}

// parse_pocket (io.cpp:162-206) of a text: 0 and the pocket (field_out gets min(cap, n) values),
// or 8 with ref_last_error() (ParseError / RangeError text).
int ref_parse_pocket(const char* text, uint64_t len, uint32_t dims[3], double origin[3], double* spacing,
                     double* field_out, uint64_t cap) {
  try {
    std::istringstream in(std::string(text, len));
    const Pocket p = parse_pocket(in);
    for (int a = 0; a < 3; ++a) {
      dims[a] = uint32_t(p.dims[a]);
      origin[a] = a == 0 ? p.origin.x : a == 1 ? p.origin.y : p.origin.z;
    }
    *spacing = p.spacing;
    for (uint64_t v = 0; v < p.field.size() && v < cap; ++v) field_out[v] = p.field[v];
    return kOk;
  } catch (const ParseError& e) {
    return fail(e, 8);
  } catch (const std::exception& e) {
    return fail(e, kOther);
  }
}

// serialize_pocket (io.cpp:208-214) into out; returns the full length.
uint64_t ref_serialize_pocket(const uint32_t dims[3], const double origin[3], double spacing, const double* field,
                              char* out, uint64_t cap) {
  const Pocket p = make_pocket_from(dims, origin, spacing, field);
  std::ostringstream os;
  serialize_pocket(os, p);
  const std::string s = os.str();
  if (out && cap) std::memcpy(out, s.data(), std::min<uint64_t>(cap, s.size()));
  return s.size();
}

}  // extern "C"
