"""CPU: the product's host side (no GPU): C-ABI exports, generator, validation, moving sets."""
import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

import paper_1901_06229_b200 as gd
from conftest import ROOT, load_npz


def test_cabi_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "geodock_b200.h")).read()
    declared = set(re.findall(r"\b(gd_[a-z_0-9]+)\s*\(", hdr))
    assert len(declared) >= 20
    lib = ctypes.CDLL(gd.lib_path())
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing


def test_generator_bit_identical_to_reference_pins():
    pins = load_npz("unit_pins")
    assert hashlib.sha256(gd.make_pocket().field.tobytes()).hexdigest() == str(pins["pocket_sha256"])
    fine = gd.make_pocket(gd.PocketSpec(dims=(47, 47, 47), spacing=0.375))
    assert hashlib.sha256(fine.field.tobytes()).hexdigest() == str(pins["fine_sha256"])
    lib = gd.make_library(gd.LibrarySpec(64, 40, 8, 0))
    h = hashlib.sha256(b"".join(getattr(lib, k).tobytes() for k in ("xyz", "radius", "bonds", "rots")))
    assert h.hexdigest() == str(pins["lib_c2_sha256"])
    assert lib.name(7) == "lig_000007"


def test_generator_matches_oracle_port(port):
    for c, a, r, s in [(20, 32, 4, 0), (3, 120, 32, 5), (4, 1, 3, 1), (4, 2, 9, 2)]:
        x, y = gd.make_library(gd.LibrarySpec(c, a, r, s)), port.make_library(c, a, r, s)
        for k in ("xyz", "radius", "bonds", "rots", "atom_off", "bond_off", "rot_off", "name_off"):
            assert np.array_equal(getattr(x, k), getattr(y, k)), k
        assert x.names == y.names


def test_count_score_calls_closed_form():
    # docking_test.cpp:59-84
    p = gd.DockParams(n_restarts=1, rotation_steps=(1, 1, 1), num_repetitions=1, dihedral_steps=2)
    assert gd.count_score_calls(p, 0) == 1
    p = gd.DockParams(n_restarts=8, rotation_steps=(8, 8, 8), num_repetitions=3, dihedral_steps=36)
    assert gd.count_score_calls(p, 2) == 5824
    assert gd.count_score_calls(gd.DockParams(), 100) == 411136


def _lig(xyz, radius, bonds=(), rots=(), name="x"):
    return gd.Library.from_ligands([dict(name=name, xyz=np.asarray(xyz, float).reshape(-1, 3),
                                         radius=radius, bonds=list(bonds), rots=list(rots))])


BAD = [
    ([[0, 0, 0], [9, 9, 9]], [1, 1], [], []),                       # disconnected (docking_test.cpp:350-358)
    ([[0, 0, 0], [1, 0, 0]], [1, -1], [(0, 1)], []),                 # non-positive radius
    ([[0, 0, 0], [1, 0, float("nan")]], [1, 1], [(0, 1)], []),       # non-finite
    ([[0, 0, 0], [1, 0, 0]], [1, 1], [(0, 5)], []),                  # bond out of range
    ([[0, 0, 0], [1, 0, 0]], [1, 1], [(0, 1), (1, 1)], []),          # self bond
    ([[0, 0, 0], [1, 0, 0], [2, 0, 0]], [1, 1, 1], [(0, 1), (1, 2)], [(0, 2)]),          # not a bond
    ([[0, 0, 0], [1, 0, 0], [1, 1, 0]], [1, 1, 1], [(0, 1), (1, 2), (2, 0)], [(0, 1)]),  # ring bond
    ([[0, 0, 0], [1, 0, 0]], [1, 1], [(0, 1)], [(0, 7)]),            # rotamer index out of range
    ([], [], [], []),                                                # no atoms
]


@pytest.mark.parametrize("case", range(len(BAD)))
def test_validation_messages(case):
    xyz, rad, bonds, rots = BAD[case]
    v = gd.validate_ligand(_lig(xyz, rad, bonds, rots))
    assert v, "expected violations"


@pytest.mark.parametrize("case", range(len(BAD)))
def test_validation_matches_reference(case, reference):
    xyz, rad, bonds, rots = BAD[case]
    lib = _lig(xyz, rad, bonds, rots)
    buf = ctypes.create_string_buffer(4096)
    P = ctypes.POINTER
    x = np.ascontiguousarray(np.asarray(xyz, float).reshape(-1, 3))
    r = np.ascontiguousarray(np.asarray(rad, float))
    b = np.ascontiguousarray(np.asarray(bonds, np.uint32).reshape(-1, 2))
    ro = np.ascontiguousarray(np.asarray(rots, np.uint32).reshape(-1, 2))
    n = reference.lib.ref_validate(ctypes.c_uint32(len(r)), x.ctypes.data_as(P(ctypes.c_double)),
                                   r.ctypes.data_as(P(ctypes.c_double)), ctypes.c_uint32(len(b)),
                                   b.ctypes.data_as(P(ctypes.c_uint32)), ctypes.c_uint32(len(ro)),
                                   ro.ctypes.data_as(P(ctypes.c_uint32)), buf, ctypes.c_uint32(4096))
    want = [s for s in buf.value.decode().split("\n") if s]
    assert n == len(want)
    assert gd.validate_ligand(lib) == want


def test_make_ligand_raises_validation_error():
    with pytest.raises(gd.ValidationError, match="is invalid"):
        gd.make_ligand("bad", [((0, 0, 0), 1.0), ((9, 9, 9), 1.0)])


def test_moving_sets_match_tree_structure():
    lib = gd.make_library(gd.LibrarySpec(30, 40, 8, 3))
    for l in range(lib.n_ligands):
        lg = lib.ligand(l)
        parent = {int(c): int(p) for p, c in lg["bonds"]}
        for r, (i, j) in enumerate(lg["rots"]):
            ms = gd.moving_set(lib, l, r)
            # child subtree of j (generate.cpp:93-103): every atom whose ancestor chain hits j
            want = []
            for a in range(40):
                x = a
                while x != 0 and x != j:
                    x = parent[x]
                if x == j:
                    want.append(a)
            assert ms.tolist() == sorted(want)
            assert i not in ms


def test_moving_set_matches_reference(reference):
    lib = gd.make_library(gd.LibrarySpec(5, 16, 6, 11))
    P = ctypes.POINTER
    for l in range(5):
        lg = lib.ligand(l)
        x = np.ascontiguousarray(lg["xyz"]); rad = np.ascontiguousarray(lg["radius"])
        b = np.ascontiguousarray(lg["bonds"]); ro = np.ascontiguousarray(lg["rots"])
        for r in range(len(ro)):
            out = np.zeros(16, np.uint32)
            n = ctypes.c_uint32()
            rc = reference.lib.ref_moving_set(ctypes.c_uint32(16), x.ctypes.data_as(P(ctypes.c_double)),
                                              rad.ctypes.data_as(P(ctypes.c_double)), ctypes.c_uint32(len(b)),
                                              b.ctypes.data_as(P(ctypes.c_uint32)), ctypes.c_uint32(len(ro)),
                                              ro.ctypes.data_as(P(ctypes.c_uint32)), ctypes.c_uint32(r),
                                              out.ctypes.data_as(P(ctypes.c_uint32)), ctypes.byref(n))
            assert rc == 0
            assert gd.moving_set(lib, l, r).tolist() == out[:n.value].tolist()


def test_library_slice_roundtrip():
    lib = gd.make_library(gd.LibrarySpec(10, 12, 3, 1))
    parts = [lib.slice(0, 3), lib.slice(3, 10)]
    assert parts[0].n_ligands == 3 and parts[1].n_ligands == 7
    assert parts[1].name(0) == "lig_000003"
    assert np.array_equal(np.vstack([p.xyz for p in parts]), lib.xyz)
    assert np.array_equal(parts[1].ligand(2)["rots"], lib.ligand(5)["rots"])


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(gd.DeviceError):
        gd.Context(0)


def test_packer_graph_checks_match_reference_on_random_graphs(reference):
    """gd_host_pack's one-DFS graph checks (connectivity, bonded rotamer, bridge via low-links,
    parallel bonds counted once) give the reference validate_ligand's verdict (molecule.cpp:176-238)
    on random trees with extra ring bonds, parallel bonds and random rotamer bonds."""
    rng = np.random.default_rng(5)
    pocket = gd.make_pocket(gd.PocketSpec())
    P = ctypes.POINTER
    seen = {True: 0, False: 0}
    for _ in range(400):
        n = int(rng.integers(1, 40))
        bonds = [(int(rng.integers(0, a)), a) for a in range(1, n)]
        for _ in range(int(rng.integers(1, 3)) if rng.random() < 0.5 else 0):
            x, z = (int(v) for v in rng.integers(0, n, 2))
            if x != z:
                bonds.append((x, z))
        if n > 1 and rng.random() < 0.15:
            bonds.append(bonds[int(rng.integers(0, len(bonds)))])
        rots = []
        for _ in range(int(rng.integers(0, min(n, 8))) if n > 1 else 0):
            i, j = bonds[int(rng.integers(0, len(bonds)))]
            rots.append((i, j) if rng.random() < 0.5 else (j, i))
        xyz = rng.uniform(-3, 3, (n, 3))
        rad = np.ones(n)
        lib = _lig(xyz, rad, bonds, rots)
        b = np.ascontiguousarray(np.asarray(bonds, np.uint32).reshape(-1, 2))
        ro = np.ascontiguousarray(np.asarray(rots, np.uint32).reshape(-1, 2))
        buf = ctypes.create_string_buffer(4096)
        nv = reference.lib.ref_validate(ctypes.c_uint32(n), xyz.ctypes.data_as(P(ctypes.c_double)),
                                        rad.ctypes.data_as(P(ctypes.c_double)), ctypes.c_uint32(len(b)),
                                        b.ctypes.data_as(P(ctypes.c_uint32)), ctypes.c_uint32(len(ro)),
                                        ro.ctypes.data_as(P(ctypes.c_uint32)), buf, ctypes.c_uint32(4096))
        try:
            gd.host_pack_seconds(lib, pocket, threads=1)
            ok = True
        except gd.ValidationError:
            ok = False
        assert ok == (nv == 0), (bonds, rots, buf.value)
        seen[ok] += 1
    assert seen[True] > 50 and seen[False] > 30
