"""GPU parity against the unmodified reference, live, on randomised instances that cover every
branch of the fast path: K1a's quarter-turn, separable and generic rotation sweeps (rotation grids
with alpha steps 16 / 8 / 12 / 10 / 6 / 24 / 32), twin frames (beta = 0 / pi rows), one-atom and
leaf-only ligands, the three size classes (<= 32, <= 64, <= 128 atoms) and the FP64 kernel
beyond, dihedral steps from 1 to 70 (S outside [2, 64] goes to the FP64 kernel), clash factors
from 0.05 (many commits) to 1, 0 to 3 repetitions, random pockets (dims 8..20 per axis, spacing
0.35..1.0, random origin).

The reference is the one compiled from /root/reference's sources by oracle/Makefile
(oracle/_ref/libgeodock_ref.so, built in this container and shipped with the snapshot); every
output and decision-trace field must match bit for bit (docking_test.cpp:322-338, acceptance #2,
acceptance_main.cpp:100-165).
"""
import numpy as np
import pytest

import paper_1901_06229_b200 as gd

pytestmark = pytest.mark.gpu

GRIDS = [(16, 16, 8), (8, 8, 4), (12, 6, 6), (10, 5, 4), (6, 6, 4), (24, 8, 4), (32, 8, 8), (16, 4, 2), (8, 3, 2)]
FIELDS = [("best_score", "best_score"), ("best_restart", "best_restart"), ("final_xyz", "final_xyz"),
          ("final_dihedrals", "final_dih"), ("align_index", "align_index"), ("step_k", "step_k"),
          ("score_calls", "score_calls")]


def _instance(rng):
    dims = tuple(int(x) for x in rng.integers(8, 21, 3))
    pocket = gd.make_pocket(gd.PocketSpec(dims=dims, spacing=float(rng.uniform(0.35, 1.0)),
                                          origin=tuple(float(x) for x in rng.uniform(-4, 4, 3)),
                                          blobs=int(rng.integers(3, 8)), seed=int(rng.integers(0, 2**62))))
    kind = rng.random()
    atoms = int(rng.integers(1, 4)) if kind < 0.1 else int(rng.integers(4, 33)) if kind < 0.55 else \
        int(rng.integers(33, 65)) if kind < 0.8 else int(rng.integers(65, 129)) if kind < 0.95 else \
        int(rng.integers(129, 180))
    rots = int(rng.integers(0, min(atoms - 1, 12) + 1)) if atoms > 1 else 0
    lib = gd.make_library(gd.LibrarySpec(int(rng.integers(1, 4)), atoms, rots, int(rng.integers(0, 2**62))))
    S = int(rng.choice([1, 2, 6, 12, 36, 70])) if rng.random() < 0.3 else int(rng.integers(2, 41))
    params = gd.DockParams(n_restarts=int(rng.integers(1, 7)), num_repetitions=int(rng.integers(0, 4)),
                           rotation_steps=GRIDS[int(rng.integers(0, len(GRIDS)))], dihedral_steps=S,
                           clash_factor=float(rng.choice([0.05, 0.1, 0.2, 0.3, 0.5, 0.75, 1.0])),
                           seed=int(rng.integers(0, 2**62)))
    return pocket, lib, params


@pytest.mark.parametrize("block", range(8))
def test_random_instances_match_live_reference(reference, block):
    from oracle import Params
    rng = np.random.default_rng(1901_06229 + block)
    ctx = gd.Context(0, mode=gd.MODE_FAST)
    try:
        for i in range(40):
            pocket, lib, p = _instance(rng)
            out = ctx.dock(lib, pocket, p, trace=True)
            ref = reference.dock(lib, pocket, Params(**p.__dict__), trace=True)
            for k_out, k_ref in FIELDS:
                assert np.array_equal(getattr(out, k_out), getattr(ref, k_ref)), (block, i, k_out, p, lib.n_ligands,
                                                                                   int(lib.atom_off[1]))
    finally:
        ctx.close()
