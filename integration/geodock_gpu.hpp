// Drop-in GPU implementations of the reference's hot-path entry points, with the reference's exact
// C++ signatures and value types (include/geodock/{docking,pipeline}.hpp in /root/reference/proj).
// A maintainer switches a caller from geodock::dock_ligand to geodock::gpu::dock_ligand (or links
// this file in place of the CPU bodies); see INTEGRATION.md. Everything below the signatures goes
// through the C-ABI in include/geodock_b200.h.
#pragma once

#include <utility>
#include <vector>

#include "geodock/docking.hpp"
#include "geodock/pipeline.hpp"

namespace geodock::gpu {

/// dock_ligand (docking.hpp:140-141): same inputs, same DockResult bits, same exceptions
/// (ValidationError / ContractError / DegenerateAxisError); runs on CUDA device 0.
DockResult dock_ligand(const Ligand& ligand, const Pocket& pocket, const DockParams& params,
                       DockStats* stats = nullptr);

/// run_screening (pipeline.hpp:85-89): the library is cut into config.n_devices contiguous
/// shards (at least one), one host thread per shard, shard d on CUDA device d % (visible devices)
/// (the reference's lanes are logical); results in library order, bit-identical for any device
/// count. n_workers and lane_width keep their ContractErrors (< 1) but otherwise have no GPU
/// meaning; hooks are ignored (the CPU retry path of pipeline.cpp:247-251 does not exist: errors
/// propagate). Every ligand is validated (validate_ligand) before any docking.
std::pair<std::vector<DockResult>, RunMetrics> run_screening(const std::vector<Ligand>& library,
                                                             const Pocket& pocket,
                                                             const DockParams& params,
                                                             const NodeConfig& config,
                                                             const PipelineHooks& hooks = {});

}  // namespace geodock::gpu
