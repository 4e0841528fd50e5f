"""GPU parity at benchmark scale and the chunked executor.

The exact kernel (GD_MODE_EXACT: the reference's FP64 arithmetic everywhere, pinned to the oracle
by test_gpu_parity.py) is the checker for the fast two-stage kernels on library sizes the CPU
oracle cannot cover in seconds: every decision and every output bit must agree. Library sizes
exceed the executor's chunk (256 ligands), so gd_dock_batch runs several pipelined chunks.
"""
import numpy as np
import pytest

import paper_1901_06229_b200 as gd

pytestmark = pytest.mark.gpu

FIELDS = ("best_score", "best_restart", "final_xyz", "final_dihedrals", "align_index", "align_score",
          "restart_score", "step_k", "score_calls")


@pytest.fixture(scope="module")
def pair():
    fast, exact = gd.Context(0, mode=gd.MODE_FAST), gd.Context(0, mode=gd.MODE_EXACT)
    yield fast, exact
    fast.close()
    exact.close()


def _same(a, b):
    for k in FIELDS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


@pytest.mark.parametrize("count,atoms,rots,clash,grid", [
    (1200, 40, 8, 0.75, None),            # C2 shape, the headline parameters
    (1200, 40, 8, 0.1, None),             # C2 shape, commits live
    (160, 120, 32, 0.75, None),           # C4 shape (NS = 4 kernels, cells from L1/L2 in K1b)
    (160, 120, 32, 0.1, None),
    (600, 40, 8, 0.3, ((47, 47, 47), 0.375)),  # C5 fine grid (cells do not fit shared memory)
])
def test_fast_equals_exact_at_scale(pair, count, atoms, rots, clash, grid):
    fast, exact = pair
    pocket = gd.make_pocket(gd.PocketSpec(dims=grid[0], spacing=grid[1]) if grid else gd.PocketSpec())
    lib = gd.make_library(gd.LibrarySpec(count, atoms, rots, 5))
    p = gd.DockParams(clash_factor=clash)
    out = fast.dock(lib, pocket, p, trace=True)
    st = fast.stats()
    _same(out, exact.dock(lib, pocket, p, trace=True))
    assert st["restarts"] == count * p.n_restarts, st


def test_second_pass_on_plateau(pair):
    """A field clamped to 1.0 over the whole box (the reference clamps its blobs to [0, 1],
    generate.cpp:44-64): every rotation that keeps the ligand inside ties exactly, so K1a's lanes
    overflow their top-4, collect every candidate in a second pass (with the twin rotations of the
    folded frames), overflow the 64-entry list and hand the restart to the FP64 alignment. The
    argmax is the lowest such index (docking.cpp:84), as in the all-FP64 kernel."""
    fast, exact = pair
    n = 24
    field = np.ones(n ** 3)
    pocket = gd.Pocket((n, n, n), (0.0, 0.0, 0.0), 0.75, field)
    lib = gd.make_library(gd.LibrarySpec(40, 12, 3, 9))
    p = gd.DockParams(n_restarts=8, clash_factor=0.3)
    out = fast.dock(lib, pocket, p, trace=True)
    st = fast.stats()
    assert st["align_second_passes"] > 0, st
    _same(out, exact.dock(lib, pocket, p, trace=True))


def test_executor_chunks_match_staged_run(pair):
    """gd_dock_batch (chunked, two streams) == gd_stage/gd_run/gd_fetch (one batch), bit for bit."""
    fast, _ = pair
    pocket = gd.make_pocket()
    lib = gd.make_library(gd.LibrarySpec(1100, 28, 5, 3))
    p = gd.DockParams(n_restarts=8, clash_factor=0.2)
    a = fast.dock(lib, pocket, p, trace=True)
    b = fast.stage(lib)
    b.run()
    c = b.fetch(trace=True)
    b.free()
    _same(a, c)
    # and again through the same (now warm, grow-only) staging slots with a different size
    _same(fast.dock(lib.slice(100, 900), pocket, p, trace=True), fast.dock(lib.slice(100, 900), pocket, p, trace=True))


def test_executor_reports_first_invalid_ligand_in_a_late_chunk(pair):
    fast, _ = pair
    good = gd.make_library(gd.LibrarySpec(700, 12, 2, 1))
    ligs = [dict(name=f"g{i}", xyz=good.xyz[good.atom_off[i]:good.atom_off[i + 1]],
                 radius=good.radius[good.atom_off[i]:good.atom_off[i + 1]],
                 bonds=good.bonds[good.bond_off[i]:good.bond_off[i + 1]],
                 rots=good.rots[good.rot_off[i]:good.rot_off[i + 1]]) for i in range(700)]
    ligs[650] = dict(name="late_bad", xyz=[[0, 0, 0], [9, 9, 9]], radius=[1.0, 1.0])
    ligs[690] = dict(name="later_bad", xyz=[[0, 0, 0]], radius=[-1.0])
    lib = gd.Library.from_ligands(ligs)
    with pytest.raises(gd.ValidationError, match="ligand 'late_bad' is invalid"):
        fast.dock(lib, gd.make_pocket(), gd.DockParams(n_restarts=2))
    # the context recovers
    out = fast.dock(lib.slice(0, 300), gd.make_pocket(), gd.DockParams(n_restarts=2))
    assert out.best_score.shape == (300,)


def test_profile_table_matches_reference_counters(pair, reference=None):
    """The profile subcommand's counters (geodock_main.cpp:189-232): DockStats closed forms."""
    fast, _ = pair
    lib = gd.make_library(gd.LibrarySpec(20, 32, 4, 0))
    p = gd.DockParams(n_restarts=8)
    prof = fast.profile(lib, gd.make_pocket(), p)
    G, R = 16 * 16 * 8, int(lib.rot_off[-1])
    assert prof["score_pose[align]"] == 8 * G * 20 and prof["score_pose[optimize]"] == 8 * 3 * R * 36
    assert prof["bump_check"] == 8 * 3 * R * 36 and prof["rotate_fragment"] == 8 * 3 * R * 35
    assert prof["total_score_calls"] == prof["expected_score_calls"]
    assert abs(prof["align_ligand"]["time_pct"] + prof["optimize_pose"]["time_pct"] - 100.0) < 1e-6
    text = gd.Context.format_profile(prof)
    assert text.splitlines()[0] == "function time_pct visits" and "expected_score_calls" in text


def _interleaved(*libs):
    """One library whose ligands alternate between the given libraries (through the .lgd text)."""
    parts = []
    for i in range(max(l.n_ligands for l in libs)):
        parts += [l.slice(i, i + 1) for l in libs if i < l.n_ligands]
    return gd.parse_library("".join(gd.serialize_library(p) for p in parts).encode())


@pytest.mark.parametrize("clash", [0.75, 0.2])
def test_mixed_sizes_route_per_ligand(pair, clash):
    """A batch mixing every size class: one fast K1a + K1b pair per class (n <= 32, <= 64, <= 128,
    NS from that class only) and the FP64 kernel for the ligands beyond 128 atoms, in one batch."""
    fast, exact = pair
    lib = _interleaved(gd.make_library(gd.LibrarySpec(40, 24, 4, 1)),    # NS = 1 class
                       gd.make_library(gd.LibrarySpec(6, 150, 6, 2)),    # FP64 kernel
                       gd.make_library(gd.LibrarySpec(20, 70, 10, 3)),   # NS = 4 class
                       gd.make_library(gd.LibrarySpec(30, 40, 8, 4)))    # NS = 2 class
    pocket = gd.make_pocket()
    p = gd.DockParams(n_restarts=8, clash_factor=clash)
    out = fast.dock(lib, pocket, p, trace=True)
    st = fast.stats()
    _same(out, exact.dock(lib, pocket, p, trace=True))
    assert st["restarts"] == 8 * lib.n_ligands  # every item exactly once across the two kernels


def test_only_large_ligands(pair):
    """Every ligand beyond 128 atoms: K1a (NS = 8) hands its candidates to the FP64 kernel."""
    fast, exact = pair
    lib = gd.make_library(gd.LibrarySpec(3, 200, 5, 8))
    pocket = gd.make_pocket()
    p = gd.DockParams(n_restarts=6, clash_factor=0.3)
    out = fast.dock(lib, pocket, p, trace=True)
    assert fast.stats()["align_exact_evals"] == 0  # (the FP64 kernel does not count candidates)
    _same(out, exact.dock(lib, pocket, p, trace=True))


@pytest.mark.parametrize("grid", [None, ((47, 47, 47), 0.375)], ids=["cells_in_smem", "cells_in_l1"])
def test_item_order_does_not_change_results(pair, grid, monkeypatch):
    """The fast kernels claim items in Morton order of the start targets where K1a reads the cells
    through L1 (C5-size grids), in ligand order where they fit shared memory; GD_NATURAL_ORDER=1
    forces ligand order. Every output and decision bit is independent of the claim order."""
    fast, _ = pair
    pocket = gd.make_pocket(gd.PocketSpec(dims=grid[0], spacing=grid[1]) if grid else gd.PocketSpec())
    lib = gd.make_library(gd.LibrarySpec(500, 40, 8, 17))
    p = gd.DockParams(clash_factor=0.1)
    chosen = fast.dock(lib, pocket, p, trace=True)
    launches = fast.stats()["launches"]
    monkeypatch.setenv("GD_NATURAL_ORDER", "1")
    natural = fast.dock(lib, pocket, p, trace=True)
    # the Morton order costs one key kernel: present on the L1 grid only
    assert launches == fast.stats()["launches"] + (1 if grid else 0)
    _same(chosen, natural)
