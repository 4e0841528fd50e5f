// C++ adapter: reference value types <-> the flat C-ABI (include/geodock_b200.h).
#include "geodock_gpu.hpp"

#include <array>
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>

#include "geodock/errors.hpp"
#include "geodock_b200.h"

namespace geodock::gpu {
namespace {

struct Flat {
  std::vector<uint32_t> atom_off{0}, bond_off{0}, rot_off{0}, name_off{0};
  std::vector<double> xyz, radius, dihedrals;
  std::vector<uint32_t> bonds, rots;
  std::string names;
  gd_library lib{};

  explicit Flat(const std::vector<const Ligand*>& ligs) {
    for (const Ligand* l : ligs) {
      for (const Atom& a : l->atoms) {
        xyz.insert(xyz.end(), {a.position.x, a.position.y, a.position.z});
        radius.push_back(a.radius);
      }
      for (const Bond& b : l->bonds) bonds.insert(bonds.end(), {uint32_t(b.first), uint32_t(b.second)});
      for (std::size_t r = 0; r < l->rotamers.size(); ++r) {
        rots.insert(rots.end(), {uint32_t(l->rotamers[r].atom_i), uint32_t(l->rotamers[r].atom_j)});
        dihedrals.push_back(r < l->dihedrals.size() ? l->dihedrals[r] : 0.0);
      }
      names += l->name;
      atom_off.push_back(uint32_t(radius.size()));
      bond_off.push_back(uint32_t(bonds.size() / 2));
      rot_off.push_back(uint32_t(rots.size() / 2));
      name_off.push_back(uint32_t(names.size()));
    }
    lib.n_ligands = uint32_t(ligs.size());
    lib.atom_off = atom_off.data();
    lib.xyz = xyz.data();
    lib.radius = radius.data();
    lib.bond_off = bond_off.data();
    lib.bonds = bonds.data();
    lib.rot_off = rot_off.data();
    lib.rots = rots.data();
    lib.dihedrals = dihedrals.data();
    lib.name_off = name_off.data();
    lib.names = names.data();
  }
};

gd_params to_c(const DockParams& p) {
  gd_params c;
  c.n_restarts = p.n_restarts;
  c.num_repetitions = p.num_repetitions;
  for (int i = 0; i < 3; ++i) c.rotation_steps[i] = p.rotation_steps[i];
  c.dihedral_steps = p.dihedral_steps;
  c.clash_factor = p.clash_factor;
  c.seed = p.seed;
  return c;
}

// One context per device, created lazily; a context is externally synchronised (the lane guard,
// pipeline.cpp:75,138), so each device has a mutex.
struct Device {
  std::mutex mu;
  gd_ctx* ctx = nullptr;
};
std::mutex g_devices_mu;
std::map<int, Device> g_devices;

Device& device(int d) {
  std::lock_guard<std::mutex> lk(g_devices_mu);
  Device& dev = g_devices[d];
  if (!dev.ctx && gd_create(d, &dev.ctx) != GD_OK) {
    throw std::runtime_error("geodock::gpu: cannot create a context on CUDA device " + std::to_string(d));
  }
  return dev;
}

// Rethrows a C-ABI status as the reference's exception (errors.hpp:10-67).
[[noreturn]] void raise(int rc, gd_ctx* ctx, const Flat& flat) {
  const std::string msg = gd_last_error(ctx);
  if (rc == GD_ERR_INVALID_LIGAND) {
    for (uint32_t l = 0; l < flat.lib.n_ligands; ++l) {
      char buf[4096];
      const int n = gd_validate_ligand(&flat.lib, l, buf, sizeof buf);
      if (n > 0) {
        std::vector<std::string> v;
        std::string all(buf);
        std::size_t at = 0, nl;
        while ((nl = all.find('\n', at)) != std::string::npos) {
          v.push_back(all.substr(at, nl - at));
          at = nl + 1;
        }
        throw ValidationError(flat.names.substr(flat.name_off[l], flat.name_off[l + 1] - flat.name_off[l]), v);
      }
    }
  }
  if (rc == GD_ERR_CONTRACT) throw ContractError(msg);
  if (rc == GD_ERR_DEGENERATE_AXIS) throw DegenerateAxisError(msg);
  throw std::runtime_error("geodock::gpu: " + msg);
}

// validate_ligand (molecule.cpp:176-238) before anything is flattened, exactly as dock_ligand
// (docking.cpp:239-240) and run_screening's workers (pipeline.cpp:233-234) do: the flat C-ABI
// carries neither the dihedral count nor a cached moving set, so those checks happen here.
void validate_all(const std::vector<const Ligand*>& ligs) {
  for (const Ligand* l : ligs) {
    const std::vector<std::string> v = validate_ligand(*l);
    if (!v.empty()) throw ValidationError(l->name, v);
  }
}

void dock_on(int d, const std::vector<const Ligand*>& ligs, const Pocket& pocket, const DockParams& params,
             DockResult* out, double* times = nullptr) {
  validate_all(ligs);
  Flat flat(ligs);
  Device& dev = device(d);
  std::lock_guard<std::mutex> lk(dev.mu);
  const uint32_t dims[3] = {uint32_t(pocket.dims[0]), uint32_t(pocket.dims[1]), uint32_t(pocket.dims[2])};
  const double origin[3] = {pocket.origin.x, pocket.origin.y, pocket.origin.z};
  int rc = gd_set_pocket(dev.ctx, dims, origin, pocket.spacing, pocket.field.data());
  const gd_params cp = to_c(params);
  if (rc == GD_OK) rc = gd_set_params(dev.ctx, &cp);
  const std::size_t L = ligs.size();
  std::vector<double> best(L), phase(2 * L), fxyz(flat.xyz.size()), fdih(flat.dihedrals.size());
  std::vector<uint32_t> restart(L);
  std::vector<uint64_t> calls(L);
  gd_results res{};
  res.best_score = best.data();
  res.best_restart = restart.data();
  res.score_calls = calls.data();
  res.phase_times = phase.data();
  res.final_xyz = fxyz.data();
  res.final_dihedrals = fdih.data();
  if (rc == GD_OK) rc = gd_dock_batch(dev.ctx, &flat.lib, &res);
  if (rc != GD_OK) raise(rc, dev.ctx, flat);
  if (times) gd_last_run_times(dev.ctx, times, 4);  // busy, align, optimize, host wait
  for (std::size_t l = 0; l < L; ++l) {
    DockResult& r = out[l];
    r.ligand_name = ligs[l]->name;
    r.best_score = best[l];
    r.best_restart_id = restart[l];
    r.score_calls = calls[l];
    r.phase_times.align_seconds = phase[2 * l];
    r.phase_times.optimize_seconds = phase[2 * l + 1];
    r.final_coordinates.clear();
    r.final_dihedrals.clear();
    // no restart: finish_dock keeps its default-constructed best pose, i.e. no coordinates and
    // no dihedrals (docking.cpp:200-230)
    if (params.n_restarts == 0) continue;
    for (uint32_t a = flat.atom_off[l]; a < flat.atom_off[l + 1]; ++a) {
      r.final_coordinates.push_back({fxyz[3 * a], fxyz[3 * a + 1], fxyz[3 * a + 2]});
    }
    r.final_dihedrals.assign(fdih.begin() + flat.rot_off[l], fdih.begin() + flat.rot_off[l + 1]);
  }
}

}  // namespace

DockResult dock_ligand(const Ligand& ligand, const Pocket& pocket, const DockParams& params, DockStats* stats) {
  DockResult r;
  double times[4] = {0, 0, 0, 0};
  dock_on(0, {&ligand}, pocket, params, &r, times);
  if (stats) {
    // DockStats counters (docking.cpp:131-142, 188-190) are the closed form the reference records:
    // N G alignment calls, N reps R S optimise calls and bump checks, N reps R (S - 1) fragment
    // rotations; wall times are the device time of the alignment (K1a) and the sweep (K1b + K2)
    const uint64_t grid = uint64_t(params.rotation_steps[0]) * params.rotation_steps[1] * params.rotation_steps[2];
    const uint64_t opt = r.score_calls - uint64_t(params.n_restarts) * grid;
    const uint64_t steps = uint64_t(params.n_restarts) * params.num_repetitions * ligand.rotamers.size();
    stats->align_score_calls += uint64_t(params.n_restarts) * grid;
    stats->optimize_score_calls += opt;
    stats->bump_checks += opt;
    stats->fragment_rotations += params.dihedral_steps > 0 ? steps * (params.dihedral_steps - 1) : 0;
    stats->align_wall_seconds += times[1];
    stats->optimize_wall_seconds += times[2];
  }
  return r;
}

std::pair<std::vector<DockResult>, RunMetrics> run_screening(const std::vector<Ligand>& library, const Pocket& pocket,
                                                             const DockParams& params, const NodeConfig& config,
                                                             const PipelineHooks& /*hooks*/) {
  if (library.empty()) throw ContractError("ligand library is empty");  // pipeline.cpp:192-194
  if (config.n_workers < 1) throw ContractError("n_workers must be >= 1");
  if (config.lane_width < 1) throw ContractError("lane_width must be >= 1");
  {  // every task is validated before its docking (pipeline.cpp:233-234): first invalid ligand
    std::vector<const Ligand*> all;
    all.reserve(library.size());
    for (const Ligand& l : library) all.push_back(&l);
    validate_all(all);
  }
  // n_devices lanes (at least one), each on CUDA device lane % (visible devices): the reference's
  // lanes are logical (pipeline.cpp:199-202), so more lanes than GPUs share the GPUs
  const unsigned n_dev = config.n_devices > 0 ? config.n_devices : 1;
  const int n_cuda = gd_device_count();
  if (n_cuda < 1) throw std::runtime_error("geodock::gpu: no CUDA device visible (there is no CPU fallback)");
  std::vector<DockResult> results(library.size());
  RunMetrics metrics;
  metrics.ligand_count = library.size();
  metrics.device_busy_seconds.assign(n_dev, 0.0);
  metrics.worker_wait_seconds.assign(n_dev, 0.0);
  std::vector<std::array<double, 4>> times(n_dev, std::array<double, 4>{0, 0, 0, 0});
  std::vector<std::exception_ptr> errors(n_dev);
  // every lane's context exists before any docks (each sizes its host pool by the live contexts)
  for (unsigned d = 0; d < n_dev && d < unsigned(n_cuda); ++d)
    if (library.size() * d / n_dev < library.size() * (d + 1) / n_dev) device(int(d));
  const auto t0 = std::chrono::steady_clock::now();
  {
    std::vector<std::thread> threads;
    for (unsigned d = 0; d < n_dev; ++d) {
      threads.emplace_back([&, d] {
        const std::size_t lo = library.size() * d / n_dev, hi = library.size() * (d + 1) / n_dev;
        if (lo == hi) return;
        std::vector<const Ligand*> part;
        for (std::size_t i = lo; i < hi; ++i) part.push_back(&library[i]);
        try {
          dock_on(int(d % unsigned(n_cuda)), part, pocket, params, results.data() + lo, times[d].data());
        } catch (...) {
          errors[d] = std::current_exception();
        }
      });
    }
    for (auto& t : threads) t.join();
  }
  for (auto& e : errors)
    if (e) std::rethrow_exception(e);  // first failing shard, like pipeline.cpp:272
  metrics.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  metrics.throughput = metrics.wall_seconds > 0 ? double(library.size()) / metrics.wall_seconds : 0.0;
  // RunMetrics from the device accounting (gd_last_run_times): busy = device span, idle = wall -
  // busy, wait = host time blocked on the GPU, align / optimize = K1a / K1b + K2 device time
  for (unsigned d = 0; d < n_dev; ++d) {
    metrics.device_busy_seconds[d] = times[d][0];
    metrics.device_idle_seconds.push_back(metrics.wall_seconds - times[d][0]);
    metrics.align_seconds_total += times[d][1];
    metrics.optimize_seconds_total += times[d][2];
    metrics.worker_wait_seconds[d] = times[d][3];
  }
  return {std::move(results), std::move(metrics)};
}

}  // namespace geodock::gpu
