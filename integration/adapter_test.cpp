// C++ parity test of the drop-in adapter against the UNMODIFIED reference, through the reference's
// own types and test helpers (tests/testkit). Mirrors docking_test.cpp:322-338
// (MatchesReferenceOracleBitForBit), acceptance #1/#2 (acceptance_main.cpp:78-165) and the error
// contract. Built by integration/Makefile here; runs on a GPU box. Exit code 0 = all pass.
#include <cstdio>
#include <sstream>
#include <string>

#include "geodock/docking.hpp"
#include "geodock/errors.hpp"
#include "geodock/generate.hpp"
#include "geodock/io.hpp"
#include "geodock/pipeline.hpp"
#include "geodock_gpu.hpp"
#include "testkit/testkit.hpp"

using namespace geodock;

static int failures = 0;
#define CHECK(cond, what)                                   \
  do {                                                      \
    if (!(cond)) {                                          \
      ++failures;                                           \
      std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
    }                                                       \
  } while (0)

static bool same_result(const DockResult& a, const DockResult& b) {  // docking_test.cpp:42-55
  if (a.ligand_name != b.ligand_name || a.best_score != b.best_score || a.best_restart_id != b.best_restart_id ||
      a.score_calls != b.score_calls || a.phase_times.align_seconds != b.phase_times.align_seconds ||
      a.phase_times.optimize_seconds != b.phase_times.optimize_seconds ||
      a.final_coordinates.size() != b.final_coordinates.size() || a.final_dihedrals != b.final_dihedrals) {
    return false;
  }
  for (std::size_t i = 0; i < a.final_coordinates.size(); ++i)
    if (!(a.final_coordinates[i] == b.final_coordinates[i])) return false;
  return true;
}

int main() {
  // 1. random testkit instances, clash 0.75 and 0.1 (acceptance #2 shape)
  for (double clash : {0.75, 0.1}) {
    SplitMix64 rng(20250807);
    int mism = 0;
    for (int i = 0; i < 60; ++i) {
      const Pocket pocket = testkit::random_pocket(rng);
      const Ligand lig = testkit::random_ligand(rng, 10, 3);
      DockParams params;
      params.n_restarts = 1 + static_cast<unsigned>(rng.below(4));
      params.rotation_steps = {6, 6, 4};
      params.num_repetitions = 1 + static_cast<unsigned>(rng.below(2));
      params.dihedral_steps = 4 + static_cast<unsigned>(rng.below(7));
      params.clash_factor = clash;
      params.seed = rng.next();
      if (!same_result(dock_ligand(lig, pocket, params), gpu::dock_ligand(lig, pocket, params))) ++mism;
    }
    std::printf("random instances clash %.2f: %d mismatches / 60\n", clash, mism);
    CHECK(mism == 0, "random instances bit-for-bit");
  }
  // 2. default parameters on the C1 library shape (32 atoms, 4 rotamers), run_screening both sides
  {
    const Pocket pocket = make_pocket(PocketSpec{});
    LibrarySpec ls;
    ls.count = 24;
    ls.atoms = 32;
    ls.rotamers = 4;
    const std::vector<Ligand> lib = make_library(ls);
    for (double clash : {0.75, 0.1}) {
      DockParams params;
      params.clash_factor = clash;
      NodeConfig cpu;
      cpu.n_workers = 8;
      auto [ref, m0] = run_screening(lib, pocket, params, cpu);
      NodeConfig gpu_cfg;
      gpu_cfg.n_devices = 1;
      auto [got, m1] = gpu::run_screening(lib, pocket, params, gpu_cfg);
      int mism = 0;
      for (std::size_t i = 0; i < lib.size(); ++i) mism += !same_result(ref[i], got[i]);
      std::printf("run_screening C1 x24 clash %.2f: %d mismatches; cpu %.2f s, gpu %.3f s\n", clash, mism,
                  m0.wall_seconds, m1.wall_seconds);
      CHECK(mism == 0, "run_screening bit-for-bit");
      // RunMetrics from the device accounting, written by the reference's own write_metrics
      CHECK(m1.device_busy_seconds.size() == 1 && m1.device_busy_seconds[0] > 0.0 &&
                m1.align_seconds_total > 0.0 && m1.optimize_seconds_total > 0.0 &&
                m1.worker_wait_seconds.size() == 1 && m1.ligand_count == lib.size(),
            "run_screening RunMetrics");
      std::ostringstream csv;
      write_metrics(csv, m1, gpu_cfg);
      CHECK(csv.str().rfind("workers,devices,lane_width,mode,ligands,", 0) == 0, "write_metrics of GPU metrics");
    }
  }
  // 2b. degenerate parameters: no restart (default-constructed result: no pose), no repetition
  {
    const Pocket pocket = make_pocket(PocketSpec{});
    LibrarySpec ls;
    ls.count = 3;
    ls.atoms = 12;
    ls.rotamers = 3;
    const std::vector<Ligand> lib = make_library(ls);
    int mism = 0;
    for (unsigned restarts : {0u, 2u}) {
      DockParams params;
      params.n_restarts = restarts;
      params.num_repetitions = restarts ? 0u : 3u;
      for (const Ligand& lig : lib)
        if (!same_result(dock_ligand(lig, pocket, params), gpu::dock_ligand(lig, pocket, params))) ++mism;
    }
    std::printf("degenerate parameters: %d mismatches / 6\n", mism);
    CHECK(mism == 0, "n_restarts = 0 and num_repetitions = 0 bit-for-bit");
  }
  // 3. error contract (errors.hpp)
  {
    SplitMix64 rng(51);
    const Pocket pocket = testkit::random_pocket(rng);
    Ligand bad;
    bad.name = "bad";
    bad.atoms = {{{0, 0, 0}, 1.0}, {{9, 9, 9}, 1.0}};
    bool got = false;
    try {
      gpu::dock_ligand(bad, pocket, DockParams{});
    } catch (const ValidationError& e) {
      got = std::string(e.what()) == "ligand 'bad' is invalid: [bond graph is not connected]";
    }
    CHECK(got, "ValidationError");
    const Ligand lig = testkit::random_ligand(rng, 8, 3);
    DockParams p;
    p.clash_factor = 1.5;
    got = false;
    try {
      gpu::dock_ligand(lig.rotamers.empty() ? testkit::random_ligand(rng, 8, 3) : lig, pocket, p);
    } catch (const ContractError&) {
      got = true;
    }
    CHECK(got || lig.rotamers.empty(), "ContractError on clash_factor");
  }
  std::printf("%s (%d failures)\n", failures ? "ADAPTER TEST FAILED" : "ADAPTER TEST PASSED", failures);
  return failures ? 1 : 0;
}
