"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes front-end for the two parity checkers built by ``oracle/Makefile``:

* ``Oracle("port")``      -> ``oracle/liboracle.so``        (our plain-C restatement)
* ``Oracle("reference")`` -> ``oracle/_ref/libgeodock_ref.so`` (the unmodified reference + shim)

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` legs import this module. The product path (``paper_1901_06229_b200``) never does.

Both libraries take the flat library layout of ``gd_library`` (include/geodock_b200.h); any object
with those numpy attributes works (``FlatLibrary`` below, or the product's ``Library``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIBS = {
    "port": os.path.join(HERE, "liboracle.so"),
    "reference": os.path.join(HERE, "_ref", "libgeodock_ref.so"),
}
_PREFIX = {"port": "go_", "reference": "ref_"}

P = C.POINTER
u32p, u64p, f64p, i32p = P(C.c_uint32), P(C.c_uint64), P(C.c_double), P(C.c_int32)


def _ptr(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


@dataclass
class FlatLibrary:
    """Flat SoA ligand library (same field names as gd_library / the product's Library)."""
    atom_off: np.ndarray
    xyz: np.ndarray
    radius: np.ndarray
    bond_off: np.ndarray
    bonds: np.ndarray
    rot_off: np.ndarray
    rots: np.ndarray
    dihedrals: np.ndarray
    name_off: np.ndarray
    names: bytes

    @property
    def n_ligands(self) -> int:
        return len(self.atom_off) - 1

    def subset(self, idx):
        idx = list(idx)
        return FlatLibrary.from_ligands([self.ligand(i) for i in idx])

    def ligand(self, i):
        a0, a1 = self.atom_off[i], self.atom_off[i + 1]
        b0, b1 = self.bond_off[i], self.bond_off[i + 1]
        r0, r1 = self.rot_off[i], self.rot_off[i + 1]
        n0, n1 = self.name_off[i], self.name_off[i + 1]
        return dict(name=self.names[n0:n1].decode(), xyz=self.xyz[a0:a1].copy(),
                    radius=self.radius[a0:a1].copy(), bonds=self.bonds[b0:b1].copy(),
                    rots=self.rots[r0:r1].copy(), dihedrals=self.dihedrals[r0:r1].copy())

    @staticmethod
    def from_ligands(ligs):
        def off(lens):
            o = np.zeros(len(lens) + 1, np.uint32)
            o[1:] = np.cumsum(lens)
            return o
        names = [l["name"].encode() for l in ligs]
        cat = lambda key, shape, dt: (np.concatenate([np.asarray(l[key], dt).reshape(shape) for l in ligs])
                                      if ligs else np.zeros((0,) + shape[1:], dt))
        return FlatLibrary(
            atom_off=off([len(l["radius"]) for l in ligs]),
            xyz=np.ascontiguousarray(cat("xyz", (-1, 3), np.float64)),
            radius=np.ascontiguousarray(cat("radius", (-1,), np.float64)),
            bond_off=off([len(np.asarray(l["bonds"]).reshape(-1, 2)) for l in ligs]),
            bonds=np.ascontiguousarray(cat("bonds", (-1, 2), np.uint32)),
            rot_off=off([len(np.asarray(l["rots"]).reshape(-1, 2)) for l in ligs]),
            rots=np.ascontiguousarray(cat("rots", (-1, 2), np.uint32)),
            dihedrals=np.ascontiguousarray(
                np.concatenate([np.asarray(l.get("dihedrals", np.zeros(len(np.asarray(l["rots"]).reshape(-1, 2)))),
                                           np.float64) for l in ligs]) if ligs else np.zeros(0)),
            name_off=off([len(s) for s in names]),
            names=b"".join(names),
        )


@dataclass
class FlatPocket:
    dims: tuple
    origin: tuple
    spacing: float
    field: np.ndarray  # x-fastest, len = nx*ny*nz

    def field_zyx(self):
        nx, ny, nz = self.dims
        return self.field.reshape(nz, ny, nx)


@dataclass
class Params:
    """Mirror of DockParams (docking.hpp:15-22)."""
    n_restarts: int = 32
    num_repetitions: int = 3
    rotation_steps: tuple = (16, 16, 8)
    dihedral_steps: int = 36
    clash_factor: float = 0.75
    seed: int = 0


@dataclass
class DockOut:
    best_score: np.ndarray
    best_restart: np.ndarray
    score_calls: np.ndarray
    phase: np.ndarray
    final_xyz: np.ndarray
    final_dih: np.ndarray
    align_index: np.ndarray = None
    align_score: np.ndarray = None
    restart_score: np.ndarray = None
    step_k: np.ndarray = None
    step_score: np.ndarray = None


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code
        self.msg = msg


class Oracle:
    def __init__(self, kind: str = "port"):
        path = _LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle {'ref' if kind == 'reference' else 'oracle'}`")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.p = _PREFIX[kind]
        f = self._fn
        f("last_error").restype = C.c_char_p
        f("fnv1a64").restype = C.c_uint64
        f("fnv1a64").argtypes = [C.c_char_p, C.c_uint64]
        f("mix_seed").restype = C.c_uint64
        f("mix_seed").argtypes = [C.c_uint64, C.c_uint64]

    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    # ---- data formats (reference only: io.cpp through the shim)
    def parse_library(self, text: bytes) -> FlatLibrary:
        """parse_ligand_library (io.cpp:96-140); raises OracleError(8 parse / 2 validation)."""
        assert self.kind == "reference", "the port has no parser"
        f = self._fn("parse_library")
        f.argtypes = [C.c_char_p, C.c_uint64]
        self._check(f(text, len(text)))
        cnt = [C.c_uint64() for _ in range(5)]
        self._fn("parse_counts")(*[C.byref(c) for c in cnt])
        L, A, B, R, N = (c.value for c in cnt)
        lib = FlatLibrary(atom_off=np.zeros(L + 1, np.uint32), xyz=np.zeros((A, 3)), radius=np.zeros(A),
                          bond_off=np.zeros(L + 1, np.uint32), bonds=np.zeros((B, 2), np.uint32),
                          rot_off=np.zeros(L + 1, np.uint32), rots=np.zeros((R, 2), np.uint32),
                          dihedrals=np.zeros(R), name_off=np.zeros(L + 1, np.uint32), names=b"")
        names = C.create_string_buffer(max(1, N))
        u32, f64 = C.POINTER(C.c_uint32), C.POINTER(C.c_double)
        self._fn("parse_fetch")(_ptr(lib.atom_off, u32), _ptr(lib.xyz, f64), _ptr(lib.radius, f64),
                                _ptr(lib.bond_off, u32), _ptr(lib.bonds, u32), _ptr(lib.rot_off, u32),
                                _ptr(lib.rots, u32), _ptr(lib.dihedrals, f64), _ptr(lib.name_off, u32), names)
        lib.names = names.raw[:N]
        return lib

    def serialize_parsed(self) -> bytes:
        """serialize_ligand_library (io.cpp:143-160) of the last parse_library result."""
        f = self._fn("serialize_parsed")
        f.restype = C.c_uint64
        n = f(None, 0)
        buf = C.create_string_buffer(n + 1)
        f(buf, n)
        return buf.raw[:n]

    def parse_pocket(self, text: bytes, cap: int = 1 << 22):
        """parse_pocket (io.cpp:162-206) -> (dims, origin, spacing, field); OracleError(8) on error."""
        f = self._fn("parse_pocket")
        dims, origin, field = np.zeros(3, np.uint32), np.zeros(3), np.zeros(cap)
        sp = C.c_double()
        f.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_double),
                      C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_uint64]
        self._check(f(text, len(text), _ptr(dims, C.POINTER(C.c_uint32)), _ptr(origin, C.POINTER(C.c_double)),
                      C.byref(sp), _ptr(field, C.POINTER(C.c_double)), cap))
        n = int(np.prod(dims.astype(np.uint64)))
        return tuple(int(x) for x in dims), tuple(float(x) for x in origin), sp.value, field[:n].copy()

    def serialize_pocket(self, dims, origin, spacing, field) -> bytes:
        """serialize_pocket (io.cpp:208-214)."""
        f = self._fn("serialize_pocket")
        f.restype = C.c_uint64
        d, o, fl = np.asarray(dims, np.uint32), np.asarray(origin, np.float64), np.ascontiguousarray(field, np.float64)
        args = [_ptr(d, C.POINTER(C.c_uint32)), _ptr(o, C.POINTER(C.c_double)), C.c_double(spacing),
                _ptr(fl, C.POINTER(C.c_double))]
        n = f(*args, None, 0)
        buf = C.create_string_buffer(n + 1)
        f(*args, buf, n)
        return buf.raw[:n]

    def write_results(self, names: list, best_score, best_restart, score_calls, phase) -> bytes:
        """write_results (io.cpp:216-223)."""
        f = self._fn("write_results")
        f.restype = C.c_uint64
        enc = [x.encode() for x in names]
        off = np.zeros(len(enc) + 1, np.uint32)
        off[1:] = np.cumsum([len(x) for x in enc])
        u32, f64, u64 = C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.POINTER(C.c_uint64)
        args = [C.c_uint64(len(enc)), _ptr(off, u32), b"".join(enc),
                _ptr(np.ascontiguousarray(best_score, np.float64), f64),
                _ptr(np.ascontiguousarray(best_restart, np.uint32), u32),
                _ptr(np.ascontiguousarray(score_calls, np.uint64), u64),
                _ptr(np.ascontiguousarray(phase, np.float64).reshape(-1), f64)]
        n = f(*args, None, 0)
        buf = C.create_string_buffer(n + 1)
        f(*args, buf, n)
        return buf.raw[:n]

    def write_metrics(self, m, cfg) -> bytes:
        """write_metrics (io.cpp:225-245) of a RunMetrics-like `m` and NodeConfig-like `cfg`."""
        f = self._fn("write_metrics")
        f.restype = C.c_uint64
        f64 = C.POINTER(C.c_double)
        arr = lambda v: np.ascontiguousarray(np.asarray(v, np.float64).reshape(-1))
        b, i, w = arr(m.device_busy_seconds), arr(m.device_idle_seconds), arr(m.worker_wait_seconds)
        args = [C.c_uint32(cfg.n_workers), C.c_uint32(cfg.n_devices), C.c_uint32(cfg.lane_width),
                C.c_int(1 if cfg.mode == "synthetic" else 0), C.c_uint64(m.ligand_count),
                C.c_double(m.wall_seconds), C.c_double(m.throughput), _ptr(b, f64), C.c_uint32(len(b)),
                _ptr(i, f64), C.c_uint32(len(i)), _ptr(w, f64), C.c_uint32(len(w)),
                C.c_double(m.align_seconds_total), C.c_double(m.optimize_seconds_total),
                C.c_uint64(m.lane_failures), C.c_uint64(m.exclusivity_violations)]
        n = f(*args, None, 0)
        buf = C.create_string_buffer(n + 1)
        f(*args, buf, n)
        return buf.raw[:n]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._fn("last_error")().decode(errors="replace"))

    # ---- primitives
    def fnv1a64(self, s: bytes) -> int:
        return self._fn("fnv1a64")(s, len(s))

    def mix_seed(self, a: int, b: int) -> int:
        return self._fn("mix_seed")(a, b)

    def rotation_grid(self, steps):
        st = np.asarray(steps, np.uint32)
        out = np.zeros((int(np.prod(st.astype(np.uint64))), 4))
        self._check(self._fn("rotation_grid")(_ptr(st, u32p), _ptr(out, f64p)))
        return out

    def sample_field(self, pocket: FlatPocket, pts):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        out = np.zeros(len(pts))
        d = np.asarray(pocket.dims, np.uint32)
        o = np.asarray(pocket.origin, np.float64)
        self._check(self._fn("sample_field")(_ptr(d, u32p), _ptr(o, f64p), C.c_double(pocket.spacing),
                                             _ptr(pocket.field, f64p), C.c_uint64(len(pts)),
                                             _ptr(pts, f64p), _ptr(out, f64p)))
        return out

    # ---- generator (generate.cpp)
    def make_pocket(self, dims=(24, 24, 24), spacing=0.75, origin=(0.0, 0.0, 0.0), blobs=6, seed=0):
        d = np.asarray(dims, np.uint32)
        o = np.asarray(origin, np.float64)
        field = np.zeros(int(np.prod(d.astype(np.uint64))))
        self._check(self._fn("make_pocket")(_ptr(d, u32p), C.c_double(spacing), _ptr(o, f64p),
                                            C.c_uint32(blobs), C.c_uint64(seed), _ptr(field, f64p)))
        return FlatPocket(tuple(int(x) for x in dims), tuple(float(x) for x in origin), float(spacing), field)

    def make_library(self, count=100, atoms=16, rotamers=4, seed=0) -> FlatLibrary:
        n = max(1, atoms)
        nr = min(rotamers, n - 1)
        xyz = np.zeros((count * n, 3))
        rad = np.zeros(count * n)
        bonds = np.zeros((count * (n - 1), 2), np.uint32)
        rots = np.zeros((count * nr, 2), np.uint32)
        self._check(self._fn("make_library")(C.c_uint64(count), C.c_uint64(atoms), C.c_uint64(rotamers),
                                             C.c_uint64(seed), _ptr(xyz, f64p), _ptr(rad, f64p),
                                             _ptr(bonds, u32p), _ptr(rots, u32p)))
        names = [b"lig_%06d" % i for i in range(count)]
        off = lambda k: np.arange(count + 1, dtype=np.uint32) * k
        noff = np.zeros(count + 1, np.uint32)
        noff[1:] = np.cumsum([len(s) for s in names])
        return FlatLibrary(off(n), xyz, rad, off(n - 1), bonds, off(nr), rots, np.zeros(count * nr),
                           noff, b"".join(names))

    # ---- the hot path
    def dock(self, lib, pocket: FlatPocket, params: Params = Params(), trace: bool = False) -> DockOut:
        L = lib.n_ligands
        N, reps = params.n_restarts, params.num_repetitions
        A = int(lib.atom_off[-1])
        Rt = int(lib.rot_off[-1])
        out = DockOut(np.zeros(L), np.zeros(L, np.uint32), np.zeros(L, np.uint64), np.zeros(2 * L),
                      np.zeros((A, 3)), np.zeros(Rt))
        if trace:
            out.align_index = np.zeros(L * N, np.uint32)
            out.align_score = np.zeros(L * N)
            out.restart_score = np.zeros(L * N)
            out.step_k = np.full(Rt * N * reps, -2, np.int32)
            out.step_score = np.zeros(Rt * N * reps)
        d = np.asarray(pocket.dims, np.uint32)
        o = np.asarray(pocket.origin, np.float64)
        st = np.asarray(params.rotation_steps, np.uint32)
        c = lambda a: np.ascontiguousarray(a)
        self._check(self._fn("dock_library")(
            C.c_uint32(L), _ptr(c(lib.atom_off), u32p), _ptr(c(lib.xyz), f64p), _ptr(c(lib.radius), f64p),
            _ptr(c(lib.bond_off), u32p), _ptr(c(lib.bonds), u32p), _ptr(c(lib.rot_off), u32p),
            _ptr(c(lib.rots), u32p), _ptr(c(lib.dihedrals), f64p), _ptr(c(lib.name_off), u32p),
            C.c_char_p(lib.names), _ptr(d, u32p), _ptr(o, f64p), C.c_double(pocket.spacing),
            _ptr(pocket.field, f64p), C.c_uint32(N), C.c_uint32(reps), _ptr(st, u32p),
            C.c_uint32(params.dihedral_steps), C.c_double(params.clash_factor), C.c_uint64(params.seed),
            _ptr(out.best_score, f64p), _ptr(out.best_restart, u32p), _ptr(out.score_calls, u64p),
            _ptr(out.phase, f64p), _ptr(out.final_xyz, f64p), _ptr(out.final_dih, f64p),
            _ptr(out.align_index, u32p), _ptr(out.align_score, f64p), _ptr(out.restart_score, f64p),
            _ptr(out.step_k, i32p), _ptr(out.step_score, f64p)))
        return out

    # ---- reference-only entry points
    def run_screening(self, lib, pocket: FlatPocket, params: Params = Params(), n_workers: int = 1):
        """The reference's production CPU path (pipeline.cpp:187-290), n_devices=0."""
        assert self.kind == "reference"
        L = lib.n_ligands
        best = np.zeros(L)
        rid = np.zeros(L, np.uint32)
        wall = C.c_double(0)
        d = np.asarray(pocket.dims, np.uint32)
        o = np.asarray(pocket.origin, np.float64)
        st = np.asarray(params.rotation_steps, np.uint32)
        c = lambda a: np.ascontiguousarray(a)
        self._check(self.lib.ref_run_screening(
            C.c_uint32(L), _ptr(c(lib.atom_off), u32p), _ptr(c(lib.xyz), f64p), _ptr(c(lib.radius), f64p),
            _ptr(c(lib.bond_off), u32p), _ptr(c(lib.bonds), u32p), _ptr(c(lib.rot_off), u32p),
            _ptr(c(lib.rots), u32p), _ptr(c(lib.name_off), u32p), C.c_char_p(lib.names),
            _ptr(d, u32p), _ptr(o, f64p), C.c_double(pocket.spacing), _ptr(pocket.field, f64p),
            C.c_uint32(params.n_restarts), C.c_uint32(params.num_repetitions), _ptr(st, u32p),
            C.c_uint32(params.dihedral_steps), C.c_double(params.clash_factor), C.c_uint64(params.seed),
            C.c_uint32(n_workers), _ptr(best, f64p), _ptr(rid, u32p), C.byref(wall)))
        return best, rid, wall.value

    def random_ligand_spec(self, state: int, max_atoms: int, max_rotamers: int):
        """testkit::random_ligand's spec draw (testkit.cpp:236-243). Returns (state', atoms, rots, seed)."""
        assert self.kind == "reference"
        s = C.c_uint64(state)
        a, r, sd = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.lib.ref_random_ligand_spec(C.byref(s), C.c_uint64(max_atoms), C.c_uint64(max_rotamers),
                                        C.byref(a), C.byref(r), C.byref(sd))
        return s.value, a.value, r.value, sd.value


# ---------------------------------------------------------------- pure-Python SplitMix64 helpers
M64 = (1 << 64) - 1


class SplitMix64:
    """prng.hpp:11-31, for driving testkit-style random instances from Python."""

    def __init__(self, seed: int):
        self.state = seed & M64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def uniform(self, lo=None, hi=None):
        u = float(self.next() >> 11) * (2.0 ** -53)
        if lo is None:
            return u
        return lo + u * (hi - lo)

    def below(self, n: int) -> int:
        return self.next() % n if n > 0 else 0


def random_pocket_spec(rng: SplitMix64):
    """testkit::random_pocket (testkit.cpp:245-256): returns make_pocket kwargs."""
    nx, ny, nz = 8 + rng.below(8), 8 + rng.below(8), 8 + rng.below(8)
    spacing = rng.uniform(0.5, 1.0)
    origin = (rng.uniform(-4.0, 4.0), rng.uniform(-4.0, 4.0), rng.uniform(-4.0, 4.0))
    blobs = 3 + rng.below(4)
    seed = rng.next()
    return dict(dims=(nx, ny, nz), spacing=spacing, origin=origin, blobs=blobs, seed=seed)


def random_ligand_spec(rng: SplitMix64, max_atoms: int, max_rotamers: int):
    """testkit::random_ligand (testkit.cpp:236-243): returns make_library kwargs (count=1)."""
    atoms = 1 + rng.below(max_atoms)
    rots = rng.below(min(max_rotamers, atoms - 1) + 1) if atoms > 1 else 0
    return dict(count=1, atoms=atoms, rotamers=rots, seed=rng.next())
