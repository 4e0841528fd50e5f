"""GPU parity: the CUDA path through the C-ABI against the reference's golden vectors and the oracle.

The bar is bit-exact: every field of every DockResult (best score, best restart, final coordinates,
final dihedrals, score calls) and the decision trace (alignment index per restart, committed
dihedral k per step, restart scores) must equal the reference's bits.
"""
import numpy as np
import pytest

import paper_1901_06229_b200 as gd
from conftest import load_json, load_npz

pytestmark = pytest.mark.gpu

MODES = [gd.MODE_EXACT, gd.MODE_FAST]


@pytest.fixture(scope="module", params=MODES, ids=["exact", "fast"])
def ctx(request):
    c = gd.Context(0, mode=request.param)
    yield c
    c.close()


def _params(d):
    d = dict(d)
    d["rotation_steps"] = tuple(d["rotation_steps"])
    return gd.DockParams(**d)


def _check_case(ctx, case, n=None):
    g = load_npz(case)
    sp = g["spec"]
    pocket = gd.make_pocket(gd.PocketSpec(**{k: tuple(v) if isinstance(v, list) else v
                                              for k, v in sp["pocket"].items()})) if sp["pocket"] else gd.make_pocket()
    lib = gd.make_library(gd.LibrarySpec(sp["count"], sp["atoms"], sp["rotamers"], sp["lib_seed"]))
    if n is not None:
        lib = lib.slice(0, n)
    n = lib.n_ligands
    p = _params(sp["params"])
    out = ctx.dock(lib, pocket, p, trace=True)
    N, reps = p.n_restarts, p.num_repetitions
    A, Rt = int(lib.atom_off[-1]), int(lib.rot_off[-1])
    assert np.array_equal(out.align_index, g["align_index"][:n * N]), "alignment decisions"
    assert np.array_equal(out.align_score, g["align_score"][:n * N]), "alignment scores"
    assert np.array_equal(out.step_k, g["step_k"][:Rt * N * reps]), "dihedral decisions"
    assert np.array_equal(out.restart_score, g["restart_score"][:n * N]), "restart scores"
    assert np.array_equal(out.best_score, g["best_score"][:n])
    assert np.array_equal(out.best_restart, g["best_restart"][:n])
    assert np.array_equal(out.final_xyz, g["final_xyz"][:A])
    assert np.array_equal(out.final_dihedrals, g["final_dih"][:Rt])
    assert np.array_equal(out.score_calls, g["score_calls"][:n])
    assert np.array_equal(out.phase_times, g["phase"][:2 * n])
    return out


@pytest.mark.parametrize("case", ["c1_default", "c1_clash01", "c2_prefix_default", "c2_prefix_clash01",
                                  "c4_prefix_clash01", "c5_prefix_default"])
def test_golden_cases_bit_exact(ctx, case):
    _check_case(ctx, case)


@pytest.mark.parametrize("case", ["random_clash075", "random_clash03"])
def test_random_instances_bit_exact(ctx, case):
    """acceptance #2 style: random pockets, ligands (<=10 atoms, <=3 rotamers) and parameters."""
    for i, row in enumerate(load_json(case)):
        pocket = gd.make_pocket(gd.PocketSpec(**{k: tuple(v) if isinstance(v, list) else v
                                                 for k, v in row["pocket"].items()}))
        lib = gd.make_library(gd.LibrarySpec(**row["ligand"]))
        out = ctx.dock(lib, pocket, _params(row["params"]), trace=True)
        assert out.best_score[0] == float.fromhex(row["best_score"]), i
        assert int(out.best_restart[0]) == row["best_restart"], i
        assert [float(x).hex() for x in out.final_xyz.ravel()] == row["final_xyz"], i
        assert [float(x).hex() for x in out.final_dihedrals] == row["final_dih"], i
        assert out.align_index.tolist() == row["align_index"], i
        assert out.step_k.tolist() == row["step_k"], i
        assert int(out.score_calls[0]) == row["score_calls"], i


def test_live_oracle_c2_prefix(ctx, port):
    """64 ligands of the C2 shape (40 atoms, 8 rotamers) at clash 0.1 against the oracle, live."""
    pocket = gd.make_pocket()
    lib = gd.make_library(gd.LibrarySpec(64, 40, 8, 0))
    p = gd.DockParams(clash_factor=0.1, n_restarts=8)
    out = ctx.dock(lib, pocket, p, trace=True)
    from oracle import Params
    ref = port.dock(lib, pocket, Params(n_restarts=8, clash_factor=0.1), trace=True)
    assert np.array_equal(out.align_index, ref.align_index)
    assert np.array_equal(out.step_k, ref.step_k)
    assert np.array_equal(out.best_score, ref.best_score)
    assert np.array_equal(out.final_xyz, ref.final_xyz)


def test_edge_cases_match_oracle(ctx, port):
    from oracle import Params
    pocket = gd.make_pocket(gd.PocketSpec(dims=(9, 11, 7), spacing=0.9, origin=(-2.0, 1.0, 0.5), seed=4))
    cases = [
        (gd.LibrarySpec(3, 1, 0, 1), gd.DockParams(n_restarts=3, rotation_steps=(4, 4, 2))),     # single atom
        (gd.LibrarySpec(3, 2, 1, 2), gd.DockParams(n_restarts=2, rotation_steps=(1, 1, 1))),     # G = 1
        (gd.LibrarySpec(2, 33, 32, 3), gd.DockParams(n_restarts=2, dihedral_steps=2, clash_factor=0.2)),  # n > 32
        (gd.LibrarySpec(2, 70, 12, 4), gd.DockParams(n_restarts=3, num_repetitions=1, clash_factor=0.15)),
        (gd.LibrarySpec(2, 12, 4, 5), gd.DockParams(n_restarts=2, dihedral_steps=97, clash_factor=0.3)),  # S > 64
        (gd.LibrarySpec(2, 12, 4, 6), gd.DockParams(n_restarts=2, dihedral_steps=1)),
        (gd.LibrarySpec(2, 12, 4, 7), gd.DockParams(n_restarts=2, num_repetitions=0)),
    ]
    for spec, p in cases:
        lib = gd.make_library(spec)
        out = ctx.dock(lib, pocket, p, trace=True)
        ref = port.dock(lib, pocket, Params(**p.__dict__), trace=True)
        assert np.array_equal(out.best_score, ref.best_score), spec
        assert np.array_equal(out.best_restart, ref.best_restart), spec
        assert np.array_equal(out.final_xyz, ref.final_xyz), spec
        assert np.array_equal(out.final_dihedrals, ref.final_dih), spec
        assert np.array_equal(out.step_k, ref.step_k), spec


@pytest.mark.parametrize("atoms,rots", [(300, 12), (1000, 24)])
def test_large_ligands_match_oracle(ctx, port, atoms, rots):
    """The reference has no atom cap (only kMaxRotamers = 128, molecule.hpp:29). Ligands beyond
    256 atoms run the all-FP64 kernel (alignment included); in a mixed batch the others keep their
    fast kernels. Bit-exact against the oracle, including the clash-0.1 commit path."""
    from oracle import Params
    pocket = gd.make_pocket()
    small = gd.make_library(gd.LibrarySpec(3, 40, 8, 1))
    big = gd.make_library(gd.LibrarySpec(1, atoms, rots, 11))
    mid = gd.make_library(gd.LibrarySpec(1, 200, 16, 12))
    lib = gd.Library.from_ligands([small.ligand(0), big.ligand(0), small.ligand(1), mid.ligand(0), small.ligand(2)])
    p = gd.DockParams(n_restarts=2, num_repetitions=1, rotation_steps=(8, 8, 4), dihedral_steps=6, clash_factor=0.1)
    out = ctx.dock(lib, pocket, p, trace=True)
    ref = port.dock(lib, pocket, Params(**p.__dict__), trace=True)
    for k_out, k_ref in [("best_score", "best_score"), ("best_restart", "best_restart"), ("final_xyz", "final_xyz"),
                         ("final_dihedrals", "final_dih"), ("align_index", "align_index"), ("step_k", "step_k")]:
        assert np.array_equal(getattr(out, k_out), getattr(ref, k_ref)), k_out
    assert (out.step_k > 0).any()  # commits happened


def test_atom_limit_is_reported(ctx):
    big = gd.make_library(gd.LibrarySpec(1, 3585, 0, 3))
    with pytest.raises(gd.GeoDockError, match="supports up to 3584"):
        ctx.dock(big, gd.make_pocket(), gd.DockParams(n_restarts=1, rotation_steps=(1, 1, 1)))


def test_uniform_field_ties_to_lowest_index(ctx, port):
    """docking_test.cpp:138-155: on a uniform field every fully-inside orientation scores exactly 1.0,
    so the lowest such grid index must win (exact-tie handling of the argmax)."""
    n = 16
    pocket = gd.Pocket((n, n, n), (0.0, 0.0, 0.0), 1.0, np.ones(n ** 3))
    lib = gd.make_library(gd.LibrarySpec(1, 5, 0, 5))
    p = gd.DockParams(n_restarts=8, rotation_steps=(6, 4, 6))
    out = ctx.dock(lib, pocket, p, trace=True)
    from oracle import FlatPocket, Params
    ref = port.dock(lib, FlatPocket(pocket.dims, pocket.origin, 1.0, pocket.field), Params(**p.__dict__), trace=True)
    assert np.array_equal(out.align_index, ref.align_index)
    assert np.array_equal(out.align_score, ref.align_score)
    assert (out.align_score == 1.0).any()


def test_planted_dihedral_optimum(ctx, port):
    """docking_test.cpp:214-243: half-turn candidate k=2 of 4 wins (dihedral = pi)."""
    n = 9
    field = np.zeros(n ** 3)
    field[(4 * n + 3) * n + 6] = 1.0
    pocket = gd.Pocket((n, n, n), (0.0, 0.0, 0.0), 1.0, field)
    lib = gd.make_ligand("dial", [((2.0, 4.0, 4.0), 0.3), ((3.5, 4.0, 4.0), 0.3), ((5.0, 4.0, 4.0), 0.3),
                                  ((6.0, 5.0, 4.0), 0.3)], [(0, 1), (1, 2), (2, 3)], [(1, 2)])
    from oracle import Params
    p = gd.DockParams(n_restarts=3, rotation_steps=(2, 2, 2), dihedral_steps=4, clash_factor=0.5)
    out = ctx.dock(lib, pocket, p, trace=True)
    ref = port.dock(lib, pocket, Params(**p.__dict__), trace=True)
    assert np.array_equal(out.step_k, ref.step_k)
    assert np.array_equal(out.best_score, ref.best_score)
    assert np.array_equal(out.final_xyz, ref.final_xyz)


def test_errors(ctx):
    pocket = gd.make_pocket()
    bad = gd.Library.from_ligands([dict(name="bad", xyz=[[0, 0, 0], [9, 9, 9]], radius=[1.0, 1.0])])
    with pytest.raises(gd.ValidationError, match="ligand 'bad' is invalid: \\[bond graph is not connected\\]"):
        ctx.dock(bad, pocket, gd.DockParams())
    lib = gd.make_library(gd.LibrarySpec(2, 8, 2, 0))
    with pytest.raises(gd.ContractError, match="clash_factor"):
        ctx.dock(lib, pocket, gd.DockParams(clash_factor=1.5))
    with pytest.raises(gd.ContractError, match="rotation grid"):
        ctx.set_params(gd.DockParams(rotation_steps=(0, 4, 4)))
    ctx.set_params(gd.DockParams())
    degen = gd.Library.from_ligands([dict(name="degen", xyz=[[0, 0, 0], [0, 0, 0], [1.5, 0, 0]],
                                          radius=[0.5] * 3, bonds=[(0, 1), (1, 2)], rots=[(0, 1)])])
    with pytest.raises(gd.DegenerateAxisError):
        ctx.dock(degen, pocket, gd.DockParams(n_restarts=2, rotation_steps=(2, 2, 2)))
    # the context is still usable after a device-side error
    out = ctx.dock(lib, pocket, gd.DockParams(n_restarts=2, rotation_steps=(2, 2, 2)))
    assert out.best_score.shape == (2,)


def test_determinism_and_sharding(ctx):
    """acceptance #1 analogue: identical bits across runs and across shard counts."""
    pocket = gd.make_pocket()
    lib = gd.make_library(gd.LibrarySpec(40, 24, 5, 9))
    p = gd.DockParams(n_restarts=6, clash_factor=0.2)
    a = ctx.dock(lib, pocket, p, trace=True)
    b = ctx.dock(lib, pocket, p, trace=True)
    parts = [ctx.dock(lib.slice(lo, hi), pocket, p, trace=True) for lo, hi in [(0, 7), (7, 23), (23, 40)]]
    for k in ("best_score", "best_restart", "final_xyz", "final_dihedrals", "align_index", "step_k"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
        assert np.array_equal(getattr(a, k), np.concatenate([getattr(q, k) for q in parts])), k


def test_topk_matches_host_sort(ctx):
    pocket = gd.make_pocket()
    lib = gd.make_library(gd.LibrarySpec(300, 16, 3, 2))
    ctx.set_pocket(pocket)
    ctx.set_params(gd.DockParams(n_restarts=4, rotation_steps=(8, 8, 4)))
    b = ctx.stage(lib)
    b.run()
    res = b.fetch()
    hits = b.topk(50)
    order = sorted(range(300), key=lambda i: (-res.best_score[i], i))[:50]
    assert [h[1] for h in hits] == order
    assert [h[0] for h in hits] == [res.best_score[i] for i in order]
    assert [h[2] for h in hits] == [int(res.best_restart[i]) for i in order]
    b.free()


def test_dock_ligand_and_run_screening_api():
    pocket = gd.make_pocket()
    lib = gd.make_library(gd.LibrarySpec(6, 32, 4, 0))
    p = gd.DockParams(n_restarts=32)
    r = gd.dock_ligand(lib.slice(1, 2), pocket, p)
    assert r.ligand_name == "lig_000001" and r.best_score == 0.8971286237470264 and r.best_restart_id == 26
    assert r.score_calls == 79360 and r.final_coordinates.shape == (32, 3)
    res, m = gd.run_screening(lib, pocket, p, devices=[0, 0])
    assert res.best_score[1] == r.best_score and m.ligand_count == 6
    # RunMetrics (pipeline.hpp:43-72) from the device accounting, and its CSV (io.cpp:225-245)
    assert len(m.device_busy_seconds) == 2 and all(b > 0 for b in m.device_busy_seconds)
    assert all(abs(m.wall_seconds - b - i) < 1e-12 for b, i in zip(m.device_busy_seconds, m.device_idle_seconds))
    assert m.align_seconds_total > 0 and m.optimize_seconds_total > 0 and len(m.worker_wait_seconds) == 2
    csv = gd.write_metrics(m, gd.NodeConfig(2, 2)).splitlines()
    assert csv[0].startswith("workers,devices,lane_width,mode,ligands") and csv[1].startswith("2,2,8,real,6,")
