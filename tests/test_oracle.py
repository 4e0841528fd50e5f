"""CPU: the oracle restatement (oracle/geodock_oracle.c) pinned against the reference.

Pins: committed golden vectors (tests/golden, generated from the unmodified reference), the
survey's Appendix-B known answers, and — when oracle/_ref is built — live bit-for-bit comparison.
"""
import hashlib

import numpy as np
import pytest

from conftest import load_json, load_npz
from oracle import Params, SplitMix64, random_ligand_spec, random_pocket_spec


def _params(d):
    d = dict(d)
    d["rotation_steps"] = tuple(d["rotation_steps"])
    return Params(**d)


def test_prng_and_hash(port):
    # fnv1a64 / mix_seed (prng.hpp:33-46) and SplitMix64 (prng.hpp:11-31) against the Python restatement
    assert port.fnv1a64(b"") == 0xCBF29CE484222325
    g = SplitMix64(123)
    import ctypes
    st = ctypes.c_uint64(123)
    port.lib.go_splitmix_next.restype = ctypes.c_uint64
    for _ in range(5):
        assert port.lib.go_splitmix_next(ctypes.byref(st)) == g.next()


def test_rotation_grid_pins(port):
    pins = load_npz("unit_pins")
    g = port.rotation_grid((16, 16, 8))
    assert np.array_equal(g, pins["grid"])
    assert np.array_equal(port.rotation_grid((6, 5, 4)), pins["grid_small"])
    # geometry_test.cpp:103-148: identity first, 2048 entries; 1840 distinct
    assert len(g) == 2048 and tuple(g[0]) == (1.0, 0.0, 0.0, 0.0)
    assert len({tuple(r) for r in g}) < 2048  # bit-identical duplicates exist (beta = 0 row)
    assert tuple(g[1]) == tuple(g[256])


def test_generator_pins(port):
    pins = load_npz("unit_pins")
    assert hashlib.sha256(port.make_pocket().field.tobytes()).hexdigest() == str(pins["pocket_sha256"])
    fine = port.make_pocket(dims=(47, 47, 47), spacing=0.375)
    assert hashlib.sha256(fine.field.tobytes()).hexdigest() == str(pins["fine_sha256"])
    lib = port.make_library(64, 40, 8, 0)
    h = hashlib.sha256(b"".join(getattr(lib, k).tobytes() for k in ("xyz", "radius", "bonds", "rots")))
    assert h.hexdigest() == str(pins["lib_c2_sha256"])


def test_sample_field_pins(port):
    pins = load_npz("unit_pins")
    assert np.array_equal(port.sample_field(port.make_pocket(), pins["pts"]), pins["sample"])


def test_sample_field_known_values(port):
    # scoring_test.cpp:30-59 re-expressed on a 4^3 / 3^3 / 2^3 uniform pocket
    from oracle import FlatPocket
    f = np.zeros(64)
    f[(3 * 4 + 2) * 4 + 1] = 0.8125
    p = FlatPocket((4, 4, 4), (0, 0, 0), 1.0, f)
    assert port.sample_field(p, [[1, 2, 3]])[0] == 0.8125
    ones = FlatPocket((4, 4, 4), (0, 0, 0), 1.0, np.ones(64))
    v = port.sample_field(ones, [[-1, 1, 1], [1, 1, 4], [3, 3, 3]])
    assert v[0] == 0.0 and v[1] == 0.0 and v[2] > 0.0
    f2 = np.zeros(8)
    for (x, y, z) in [(1, 0, 0), (1, 1, 0), (1, 0, 1), (1, 1, 1)]:
        f2[(z * 2 + y) * 2 + x] = 1.0
    assert port.sample_field(FlatPocket((2, 2, 2), (0, 0, 0), 1.0, f2), [[0.5, 0.5, 0.5]])[0] == 0.5
    f3 = np.zeros(27)
    f3[(1 * 3 + 1) * 3 + 1] = 1.0
    assert abs(port.sample_field(FlatPocket((3, 3, 3), (0, 0, 0), 1.0, f3), [[1, 1, 1.25]])[0] - 0.75) < 1e-12


@pytest.mark.parametrize("case", ["c1_default", "c1_clash01", "c2_prefix_clash01", "c5_prefix_default"])
def test_dock_matches_golden(port, case):
    g = load_npz(case)
    sp = g["spec"]
    n = {"c1_default": 12, "c1_clash01": 12}.get(case, 4)  # prefix keeps the CPU suite fast
    pocket = port.make_pocket(**sp["pocket"]) if sp["pocket"] else port.make_pocket()
    lib = port.make_library(sp["count"], sp["atoms"], sp["rotamers"], sp["lib_seed"]).subset(range(n))
    out = port.dock(lib, pocket, _params(sp["params"]), trace=True)
    N, reps = sp["params"]["n_restarts"], sp["params"]["num_repetitions"]
    A, Rt = int(lib.atom_off[-1]), int(lib.rot_off[-1])
    assert np.array_equal(out.best_score, g["best_score"][:n])
    assert np.array_equal(out.best_restart, g["best_restart"][:n])
    assert np.array_equal(out.score_calls, g["score_calls"][:n])
    assert np.array_equal(out.final_xyz, g["final_xyz"][:A])
    assert np.array_equal(out.final_dih, g["final_dih"][:Rt])
    assert np.array_equal(out.align_index, g["align_index"][:n * N])
    assert np.array_equal(out.align_score, g["align_score"][:n * N])
    assert np.array_equal(out.restart_score, g["restart_score"][:n * N])
    assert np.array_equal(out.step_k, g["step_k"][:Rt * N * reps])


def test_appendix_b_known_answers(port):
    pocket = port.make_pocket()
    lib = port.make_library(3, 32, 4, 0)
    out = port.dock(lib, pocket, Params(), trace=True)
    assert out.best_score[0] == 0.95255757445378142 and out.best_restart[0] == 1
    assert out.best_score[1] == 0.8971286237470264 and out.best_restart[1] == 26
    assert out.best_score[2] == 0.84058791242283559 and out.best_restart[2] == 12
    assert out.align_index[0 * 32 + 1] == 1456 and out.align_index[1 * 32 + 26] == 50
    assert out.score_calls[0] == 79360
    assert out.final_xyz[0, 0] == 6.6819567129934514
    out = port.dock(lib, pocket, Params(clash_factor=0.1))
    assert out.best_score[0] == 0.95487053124515564
    assert out.best_score[1] == 0.92566237539623575


@pytest.mark.parametrize("case", ["random_clash075", "random_clash03"])
def test_random_instances_match_golden(port, case):
    for row in load_json(case)[:40]:
        pocket = port.make_pocket(**row["pocket"])
        lib = port.make_library(**row["ligand"])
        out = port.dock(lib, pocket, _params(row["params"]), trace=True)
        assert out.best_score[0] == float.fromhex(row["best_score"])
        assert int(out.best_restart[0]) == row["best_restart"]
        assert [float(x).hex() for x in out.final_xyz.ravel()] == row["final_xyz"]
        assert out.align_index.tolist() == row["align_index"]
        assert out.step_k.tolist() == row["step_k"]


def test_live_against_reference_build(port, reference):
    """Bit-for-bit, live: random testkit-style instances (acceptance_main.cpp:100-165)."""
    rng = SplitMix64(99)
    for i in range(15):
        pk = random_pocket_spec(rng)
        lk = random_ligand_spec(rng, 12, 4)
        params = Params(n_restarts=1 + rng.below(4), rotation_steps=(1 + rng.below(6), 1 + rng.below(6), 1 + rng.below(4)),
                        num_repetitions=1 + rng.below(3), dihedral_steps=2 + rng.below(9),
                        clash_factor=[0.75, 0.3, 0.1][i % 3], seed=rng.next())
        pa, pb = port.make_pocket(**pk), reference.make_pocket(**pk)
        assert np.array_equal(pa.field, pb.field)
        lib = port.make_library(**lk)
        a = port.dock(lib, pa, params, trace=True)
        b = reference.dock(lib, pb, params, trace=True)
        for k in a.__dataclass_fields__:
            assert np.array_equal(getattr(a, k), getattr(b, k)), (i, k)
