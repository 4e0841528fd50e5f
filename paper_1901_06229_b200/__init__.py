"""geodock_b200 — B200-native GeoDock pose search (arXiv 1901.06229 hot path), Python host API.

This module mirrors the reference's plugin interface for the hot path
(/root/reference/proj/include/geodock/{docking,pipeline,generate,molecule,scoring}.hpp):

    DockParams, Pocket, make_pocket(PocketSpec), make_library(LibrarySpec), make_ligand(...)
    dock_ligand(ligand, pocket, params) -> DockResult            (docking.hpp:140-141)
    run_screening(library, pocket, params, n_devices) -> (results, RunMetrics)  (pipeline.hpp:85-89)

Every docking call goes through the C-ABI in ``libgeodock_b200.so`` (include/geodock_b200.h) and
runs on the GPU. There is no CPU fallback: if the shared library or a GPU is missing, calls raise.
Errors map to the reference's exception types (errors.hpp:10-67).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
import time
import warnings
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "DockParams", "PocketSpec", "LibrarySpec", "Pocket", "Library", "DockResult", "DockResults",
    "RunMetrics", "NodeConfig", "write_metrics", "Context", "make_pocket", "make_library", "make_ligand", "dock_ligand",
    "run_screening", "count_score_calls", "validate_ligand", "moving_set", "GeoDockError",
    "ValidationError", "ContractError", "DegenerateAxisError", "DeviceError", "ParseError", "lib_path",
    "parse_library", "load_library", "serialize_library", "format_double", "write_results",
    "parse_pocket", "load_pocket", "serialize_pocket",
    "MODE_FAST", "MODE_EXACT", "FLAG_SKIP_INVARIANT_CLASH",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgeodock_b200.so")

GD_OK, GD_ERR_ARGUMENT, GD_ERR_INVALID_LIGAND, GD_ERR_CONTRACT = 0, 1, 2, 3
GD_ERR_DEGENERATE_AXIS, GD_ERR_CUDA, GD_ERR_NO_POCKET, GD_ERR_UNSUPPORTED, GD_ERR_PARSE = 4, 5, 6, 7, 8
MODE_FAST, MODE_EXACT, FLAG_SKIP_INVARIANT_CLASH = 0, 1, 0x100


# ----------------------------------------------------------------------------- errors
class GeoDockError(RuntimeError):
    code = -1


class ValidationError(GeoDockError):   # errors.hpp:37-56
    code = GD_ERR_INVALID_LIGAND


class ContractError(GeoDockError):     # errors.hpp:10-14
    code = GD_ERR_CONTRACT


class DegenerateAxisError(GeoDockError):  # errors.hpp:64-67
    code = GD_ERR_DEGENERATE_AXIS


class DeviceError(GeoDockError):
    code = GD_ERR_CUDA


class ParseError(GeoDockError):        # errors.hpp:15-27 (message carries " (line N)")
    code = GD_ERR_PARSE


_ERRORS = {GD_ERR_INVALID_LIGAND: ValidationError, GD_ERR_CONTRACT: ContractError,
           GD_ERR_DEGENERATE_AXIS: DegenerateAxisError, GD_ERR_CUDA: DeviceError, GD_ERR_PARSE: ParseError}


# ----------------------------------------------------------------------------- ctypes layer
class _Params(C.Structure):
    _fields_ = [("n_restarts", C.c_uint32), ("num_repetitions", C.c_uint32),
                ("rotation_steps", C.c_uint32 * 3), ("dihedral_steps", C.c_uint32),
                ("clash_factor", C.c_double), ("seed", C.c_uint64)]


_u32p, _u64p, _f64p, _i32p = (C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                              C.POINTER(C.c_double), C.POINTER(C.c_int32))


class _Library(C.Structure):
    _fields_ = [("n_ligands", C.c_uint32), ("atom_off", _u32p), ("xyz", _f64p), ("radius", _f64p),
                ("bond_off", _u32p), ("bonds", _u32p), ("rot_off", _u32p), ("rots", _u32p),
                ("dihedrals", _f64p), ("name_off", _u32p), ("names", C.c_char_p)]


class _Results(C.Structure):
    _fields_ = [("best_score", _f64p), ("best_restart", _u32p), ("score_calls", _u64p),
                ("phase_times", _f64p), ("final_xyz", _f64p), ("final_dihedrals", _f64p),
                ("align_index", _u32p), ("align_score", _f64p), ("restart_score", _f64p),
                ("step_k", _i32p)]


class _Hit(C.Structure):
    _fields_ = [("best_score", C.c_double), ("ligand", C.c_uint32), ("restart", C.c_uint32)]


class _Stats(C.Structure):
    _fields_ = [("restarts", C.c_uint64), ("align_exact_evals", C.c_uint64),
                ("align_fallbacks", C.c_uint64), ("step_exact_evals", C.c_uint64),
                ("step_fallbacks", C.c_uint64), ("commits", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("launches", C.c_uint32), ("exact_fallback", C.c_uint32),
                ("align_second_passes", C.c_uint64), ("sweep_steps", C.c_uint64),
                ("sweep_invariant_steps", C.c_uint64), ("sweep_scored_steps", C.c_uint64),
                ("sweep_samples", C.c_uint64), ("cross_pairs", C.c_uint64),
                ("sweep_moves", C.c_uint64), ("step_exact_score_evals", C.c_uint64),
                ("step_exact_allout_evals", C.c_uint64), ("step_exact_face_evals", C.c_uint64),
                ("step_exact_clash_evals", C.c_uint64)]


_lib = None
_lib_lock = threading.Lock()


def lib_path() -> str:
    return _LIB_PATH


def _load():
    """Loads the in-tree C-ABI library; raises if it is missing (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} not built: run `python -m paper_1901_06229_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        lib = C.CDLL(_LIB_PATH)
        vp = C.c_void_p
        sig = {
            "gd_default_params": (_Params, []),
            "gd_version": (C.c_char_p, []),
            "gd_device_count": (C.c_int, []),
            "gd_host_pack": (C.c_int, [C.POINTER(_Library), C.POINTER(_Params), _u32p, _f64p, C.c_double,
                                       C.c_uint32, C.POINTER(C.c_double)]),
            "gd_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
            "gd_destroy": (None, [vp]),
            "gd_last_error": (C.c_char_p, [vp]),
            "gd_set_pocket": (C.c_int, [vp, _u32p, _f64p, C.c_double, _f64p]),
            "gd_set_params": (C.c_int, [vp, C.POINTER(_Params)]),
            "gd_set_mode": (C.c_int, [vp, C.c_int]),
            "gd_dock_batch": (C.c_int, [vp, C.POINTER(_Library), C.POINTER(_Results)]),
            "gd_stage": (C.c_int, [vp, C.POINTER(_Library), C.POINTER(vp)]),
            "gd_run": (C.c_int, [vp]),
            "gd_fetch": (C.c_int, [vp, C.POINTER(_Results)]),
            "gd_topk": (C.c_int, [vp, C.c_uint32, C.POINTER(_Hit), _u32p]),
            "gd_batch_free": (None, [vp]),
            "gd_sync": (C.c_int, [vp]),
            "gd_stream": (vp, [vp]),
            "gd_last_stats": (C.c_int, [vp, C.POINTER(_Stats)]),
            "gd_last_kernel_ms": (C.c_int, [vp, C.POINTER(C.c_float), C.c_uint32]),
            "gd_last_run_times": (C.c_int, [vp, C.POINTER(C.c_double), C.c_uint32]),
            "gd_count_score_calls": (C.c_uint64, [C.POINTER(_Params), C.c_uint64]),
            "gd_validate_ligand": (C.c_int, [C.POINTER(_Library), C.c_uint32, C.c_char_p, C.c_uint32]),
            "gd_moving_set": (C.c_int, [C.POINTER(_Library), C.c_uint32, C.c_uint32, _u32p, _u32p]),
            "gd_make_pocket": (C.c_int, [_u32p, C.c_double, _f64p, C.c_uint32, C.c_uint64, _f64p]),
            "gd_parse_library": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(vp), C.c_char_p, C.c_uint32]),
            "gd_libbuf_view": (C.c_int, [vp, C.POINTER(_Library)]),
            "gd_libbuf_free": (None, [vp]),
            "gd_parse_pocket": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(vp), C.c_char_p, C.c_uint32]),
            "gd_pocketbuf_view": (C.c_int, [vp, _u32p, _f64p, C.POINTER(C.c_double),
                                            C.POINTER(C.POINTER(C.c_double))]),
            "gd_pocketbuf_free": (None, [vp]),
            "gd_make_library": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _f64p,
                                          _f64p, _u32p, _u32p]),
            "gd_make_library_range": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                                _f64p, _f64p, _u32p, _u32p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


# ----------------------------------------------------------------------------- value types
@dataclass
class DockParams:
    """docking.hpp:15-22."""
    n_restarts: int = 32
    num_repetitions: int = 3
    rotation_steps: Tuple[int, int, int] = (16, 16, 8)
    dihedral_steps: int = 36
    clash_factor: float = 0.75
    seed: int = 0

    def _c(self) -> _Params:
        p = _Params()
        p.n_restarts, p.num_repetitions = self.n_restarts, self.num_repetitions
        for i in range(3):
            p.rotation_steps[i] = self.rotation_steps[i]
        p.dihedral_steps, p.clash_factor, p.seed = self.dihedral_steps, self.clash_factor, self.seed
        return p


@dataclass
class PocketSpec:
    """generate.hpp:12-18."""
    dims: Tuple[int, int, int] = (24, 24, 24)
    spacing: float = 0.75
    origin: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    blobs: int = 6
    seed: int = 0


@dataclass
class LibrarySpec:
    """generate.hpp:22-28."""
    count: int = 100
    atoms: int = 16
    rotamers: int = 4
    seed: int = 0


@dataclass
class Pocket:
    """scoring.hpp:18-37: x-fastest FP64 field (index (iz*ny + iy)*nx + ix)."""
    dims: Tuple[int, int, int]
    origin: Tuple[float, float, float]
    spacing: float
    field: np.ndarray

    def bounds_lo(self):
        return tuple(self.origin)

    def bounds_hi(self):
        return tuple(o + self.spacing * float(d - 1) for o, d in zip(self.origin, self.dims))


@dataclass
class Library:
    """Flat SoA ligand library = gd_library (include/geodock_b200.h)."""
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

    def __len__(self):
        return self.n_ligands

    def name(self, i) -> str:
        return self.names[self.name_off[i]:self.name_off[i + 1]].decode()

    def n_atoms(self, i) -> int:
        return int(self.atom_off[i + 1] - self.atom_off[i])

    def n_rotamers(self, i) -> int:
        return int(self.rot_off[i + 1] - self.rot_off[i])

    def ligand(self, i) -> dict:
        a0, a1 = self.atom_off[i], self.atom_off[i + 1]
        b0, b1 = self.bond_off[i], self.bond_off[i + 1]
        r0, r1 = self.rot_off[i], self.rot_off[i + 1]
        return dict(name=self.name(i), xyz=self.xyz[a0:a1].copy(), radius=self.radius[a0:a1].copy(),
                    bonds=self.bonds[b0:b1].copy(), rots=self.rots[r0:r1].copy(),
                    dihedrals=self.dihedrals[r0:r1].copy())

    def slice(self, lo: int, hi: int) -> "Library":
        """Contiguous shard [lo, hi) with re-based offsets (for multi-GPU sharding)."""
        a0, b0, r0, n0 = (int(self.atom_off[lo]), int(self.bond_off[lo]), int(self.rot_off[lo]),
                          int(self.name_off[lo]))
        return Library(
            atom_off=(self.atom_off[lo:hi + 1] - a0).astype(np.uint32),
            xyz=self.xyz[a0:int(self.atom_off[hi])], radius=self.radius[a0:int(self.atom_off[hi])],
            bond_off=(self.bond_off[lo:hi + 1] - b0).astype(np.uint32),
            bonds=self.bonds[b0:int(self.bond_off[hi])],
            rot_off=(self.rot_off[lo:hi + 1] - r0).astype(np.uint32),
            rots=self.rots[r0:int(self.rot_off[hi])], dihedrals=self.dihedrals[r0:int(self.rot_off[hi])],
            name_off=(self.name_off[lo:hi + 1] - n0).astype(np.uint32),
            names=self.names[n0:int(self.name_off[hi])])

    def take(self, idx) -> "Library":
        """The ligands idx (any order, repeats allowed) as a new library (vectorised gather)."""
        idx = np.asarray(idx, np.int64)

        def gather(off, arr):
            lo, hi = off[idx].astype(np.int64), off[idx + 1].astype(np.int64)
            lens = hi - lo
            o = np.zeros(len(idx) + 1, np.uint32)
            o[1:] = np.cumsum(lens)
            src = np.repeat(lo - o[:-1].astype(np.int64), lens) + np.arange(int(o[-1]), dtype=np.int64)
            return o, arr[src]

        ao, xyz = gather(self.atom_off, self.xyz)
        _, rad = gather(self.atom_off, self.radius)
        bo, bonds = gather(self.bond_off, self.bonds)
        ro, rots = gather(self.rot_off, self.rots)
        _, dih = gather(self.rot_off, self.dihedrals)
        no, names = gather(self.name_off, np.frombuffer(self.names, np.uint8))
        return Library(ao, xyz, rad, bo, bonds, ro, rots, dih, no, names.tobytes())

    @staticmethod
    def from_ligands(ligs: Sequence[dict]) -> "Library":
        def off(lens):
            o = np.zeros(len(lens) + 1, np.uint32)
            if lens:
                o[1:] = np.cumsum(lens)
            return o

        def cat(key, width, dt):
            parts = [np.asarray(l.get(key, []), dt).reshape(-1, width) if width > 1 else
                     np.asarray(l.get(key, []), dt).reshape(-1) for l in ligs]
            if not parts:
                return np.zeros((0, width) if width > 1 else (0,), dt)
            return np.ascontiguousarray(np.concatenate(parts))

        names = [l["name"].encode() for l in ligs]
        rots = [np.asarray(l.get("rots", []), np.uint32).reshape(-1, 2) for l in ligs]
        dih = [np.asarray(l["dihedrals"], np.float64) if "dihedrals" in l else np.zeros(len(r))
               for l, r in zip(ligs, rots)]
        return Library(
            atom_off=off([len(np.asarray(l["radius"]).reshape(-1)) for l in ligs]),
            xyz=cat("xyz", 3, np.float64), radius=cat("radius", 1, np.float64),
            bond_off=off([len(np.asarray(l.get("bonds", []), np.uint32).reshape(-1, 2)) for l in ligs]),
            bonds=cat("bonds", 2, np.uint32),
            rot_off=off([len(r) for r in rots]), rots=cat("rots", 2, np.uint32),
            dihedrals=np.ascontiguousarray(np.concatenate(dih)) if dih else np.zeros(0),
            name_off=off([len(s) for s in names]), names=b"".join(names))

    def _c(self) -> Tuple[_Library, list]:
        keep = [np.ascontiguousarray(a) for a in (self.atom_off, self.xyz, self.radius, self.bond_off,
                                                   self.bonds, self.rot_off, self.rots, self.dihedrals,
                                                   self.name_off)]
        keep[0], keep[3], keep[5], keep[8] = (k.astype(np.uint32, copy=False) for k in
                                              (keep[0], keep[3], keep[5], keep[8]))
        keep[4], keep[6] = keep[4].astype(np.uint32, copy=False), keep[6].astype(np.uint32, copy=False)
        keep[1], keep[2], keep[7] = (k.astype(np.float64, copy=False) for k in (keep[1], keep[2], keep[7]))
        L = _Library()
        L.n_ligands = self.n_ligands
        L.atom_off, L.xyz, L.radius = _p(keep[0], _u32p), _p(keep[1], _f64p), _p(keep[2], _f64p)
        L.bond_off, L.bonds = _p(keep[3], _u32p), _p(keep[4], _u32p)
        L.rot_off, L.rots, L.dihedrals = _p(keep[5], _u32p), _p(keep[6], _u32p), _p(keep[7], _f64p)
        L.name_off, L.names = _p(keep[8], _u32p), self.names
        keep.append(self.names)
        return L, keep


@dataclass
class DockResult:
    """docking.hpp:34-42."""
    ligand_name: str
    best_score: float
    best_restart_id: int
    final_coordinates: np.ndarray
    final_dihedrals: np.ndarray
    score_calls: int
    align_seconds: float
    optimize_seconds: float


@dataclass
class DockResults:
    """Batch results (flat, library order). Trace arrays are filled when requested."""
    best_score: np.ndarray
    best_restart: np.ndarray
    score_calls: np.ndarray
    phase_times: np.ndarray
    final_xyz: np.ndarray
    final_dihedrals: np.ndarray
    align_index: Optional[np.ndarray] = None
    align_score: Optional[np.ndarray] = None
    restart_score: Optional[np.ndarray] = None
    step_k: Optional[np.ndarray] = None

    def result(self, lib: Library, i: int) -> DockResult:
        a0, a1 = int(lib.atom_off[i]), int(lib.atom_off[i + 1])
        r0, r1 = int(lib.rot_off[i]), int(lib.rot_off[i + 1])
        return DockResult(lib.name(i), float(self.best_score[i]), int(self.best_restart[i]),
                          self.final_xyz[a0:a1].copy(), self.final_dihedrals[r0:r1].copy(),
                          int(self.score_calls[i]), float(self.phase_times[2 * i]),
                          float(self.phase_times[2 * i + 1]))


@dataclass
class NodeConfig:
    """NodeConfig (pipeline.hpp:21-34) as a GPU run uses it: one host thread per GPU, no lanes
    (lane_width kept for the metrics CSV), always real mode (the synthetic scheduler is out of scope)."""
    n_workers: int = 1
    n_devices: int = 1
    lane_width: int = 8
    mode: str = "real"


@dataclass
class RunMetrics:
    """RunMetrics (pipeline.hpp:43-72) as a GPU run reports it. Per GPU: device_busy_seconds = the
    device span of its gd_dock_batch (first K1a start to last K2 end, CUDA events),
    device_idle_seconds = wall - busy, worker_wait_seconds = its host thread's time waiting on the
    GPU. align/optimize_seconds_total = device time of K1a / K1b + K2 (per-chunk event intervals,
    summed over GPUs). Offload records, claim/finish workers, lane failures and exclusivity
    violations belong to the reference's CPU-lane scheduler (no CPU retry here): empty / 0."""
    wall_seconds: float = 0.0
    throughput: float = 0.0
    ligand_count: int = 0
    device_busy_seconds: List[float] = field(default_factory=list)
    device_idle_seconds: List[float] = field(default_factory=list)
    worker_wait_seconds: List[float] = field(default_factory=list)
    align_seconds_total: float = 0.0
    optimize_seconds_total: float = 0.0
    lane_failures: int = 0
    exclusivity_violations: int = 0

    def total_wait_seconds(self) -> float:
        """RunMetrics::total_wait_seconds (pipeline.hpp:62-66)."""
        return float(sum(self.worker_wait_seconds))


# ----------------------------------------------------------------------------- host helpers
def count_score_calls(params: DockParams, n_rotamers: int) -> int:
    """docking.cpp:44-50."""
    return int(_load().gd_count_score_calls(C.byref(params._c()), n_rotamers))


def make_pocket(spec: PocketSpec = PocketSpec()) -> Pocket:
    """generate.cpp:27-66 (host, deterministic)."""
    d = np.asarray(spec.dims, np.uint32)
    o = np.asarray(spec.origin, np.float64)
    f = np.zeros(int(np.prod(d.astype(np.uint64))))
    rc = _load().gd_make_pocket(_p(d, _u32p), spec.spacing, _p(o, _f64p), spec.blobs, spec.seed, _p(f, _f64p))
    if rc:
        raise GeoDockError(f"gd_make_pocket failed ({rc})")
    return Pocket(tuple(int(x) for x in spec.dims), tuple(float(x) for x in spec.origin), float(spec.spacing), f)


def make_library(spec: LibrarySpec = LibrarySpec(), first: int = 0, count: Optional[int] = None) -> Library:
    """generate.cpp:68-109 (host, deterministic, multi-threaded). ``first``/``count`` select ligands
    [first, first + count) of the spec's library (default: all of it), e.g. one rank's shard;
    every ligand has its own random stream, so a range equals the same slice of the whole."""
    count = spec.count - first if count is None else count
    n = max(1, spec.atoms)
    nr = min(spec.rotamers, n - 1)
    xyz = np.zeros((count * n, 3))
    rad = np.zeros(count * n)
    bonds = np.zeros((count * (n - 1), 2), np.uint32)
    rots = np.zeros((count * nr, 2), np.uint32)
    rc = _load().gd_make_library_range(first, count, spec.atoms, spec.rotamers, spec.seed, _p(xyz, _f64p),
                                       _p(rad, _f64p), _p(bonds, _u32p), _p(rots, _u32p))
    if rc:
        raise GeoDockError(f"gd_make_library_range failed ({rc})")
    names = [b"lig_%06d" % i for i in range(first, first + count)]  # lig_%06zu (generate.cpp:78)
    name_off = np.zeros(count + 1, np.uint32)
    if count:
        name_off[1:] = np.cumsum([len(x) for x in names])
    ar = lambda k: (np.arange(count + 1, dtype=np.uint32) * k).astype(np.uint32)
    return Library(ar(n), xyz, rad, ar(n - 1), bonds, ar(nr), rots, np.zeros(count * nr), name_off, b"".join(names))


def make_ligand(name: str, atoms: Sequence[Tuple[Sequence[float], float]], bonds=(), rotamer_bonds=()) -> Library:
    """make_ligand (molecule.cpp:101-115): a one-ligand Library; raises ValidationError if invalid."""
    lib = Library.from_ligands([dict(name=name, xyz=[a[0] for a in atoms] or np.zeros((0, 3)),
                                     radius=[a[1] for a in atoms], bonds=list(bonds),
                                     rots=list(rotamer_bonds))])
    v = validate_ligand(lib, 0)
    if v:
        raise ValidationError(f"ligand '{name}' is invalid:" + "".join(f" [{s}]" for s in v))
    return lib


def host_pack_seconds(lib: Library, pocket: Pocket, params: DockParams = DockParams(), threads: int = 0) -> float:
    """Wall time of the executor's host half (validate + SoA pack) for `lib`, no GPU needed."""
    L, keep = lib._c()
    d = np.asarray(pocket.dims, np.uint32)
    o = np.asarray(pocket.origin, np.float64)
    t = C.c_double()
    rc = _load().gd_host_pack(C.byref(L), C.byref(params._c()), _p(d, _u32p), _p(o, _f64p), pocket.spacing,
                              threads, C.byref(t))
    if rc:
        raise _ERRORS.get(rc, GeoDockError)(f"gd_host_pack failed ({rc})")
    return t.value


def validate_ligand(lib: Library, i: int = 0) -> List[str]:
    """validate_ligand (molecule.cpp:176-238): list of violations, empty when well formed."""
    L, keep = lib._c()
    buf = C.create_string_buffer(4096)
    n = _load().gd_validate_ligand(C.byref(L), i, buf, len(buf))
    return [s for s in buf.value.decode().split("\n") if s][:max(n, 0)]


# ----------------------------------------------------------------------------- data formats
def parse_library(text) -> Library:
    """parse_ligand_library (io.cpp:96-140) over a whole .lgd text (str or bytes), multi-threaded
    in the C++ host library; every record is validated like the reference's parser does. Raises
    ParseError / ValidationError with the reference's message."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    lib = _load()
    h = C.c_void_p()
    err = C.create_string_buffer(4096)
    rc = lib.gd_parse_library(data, len(data), C.byref(h), err, len(err))
    if rc:
        raise _ERRORS.get(rc, GeoDockError)(err.value.decode(errors="replace"))
    try:
        v = _Library()
        lib.gd_libbuf_view(h, C.byref(v))
        L = v.n_ligands
        off = lambda p, n: np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.uint32)
        ao, bo, ro, no = (off(getattr(v, k), L + 1) for k in ("atom_off", "bond_off", "rot_off", "name_off"))
        A, B, R, N = int(ao[-1]), int(bo[-1]), int(ro[-1]), int(no[-1])
        arr = lambda p, n, dt: (np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, dt))
        return Library(atom_off=ao, xyz=arr(v.xyz, 3 * A, np.float64).reshape(-1, 3), radius=arr(v.radius, A, np.float64),
                       bond_off=bo, bonds=arr(v.bonds, 2 * B, np.uint32).reshape(-1, 2), rot_off=ro,
                       rots=arr(v.rots, 2 * R, np.uint32).reshape(-1, 2), dihedrals=arr(v.dihedrals, R, np.float64),
                       name_off=no, names=C.string_at(v.names, N) if N else b"")
    finally:
        lib.gd_libbuf_free(h)


def load_library(path: str) -> Library:
    """load_ligand_library (io.cpp:266-269)."""
    with open(path, "rb") as f:
        return parse_library(f.read())


def parse_pocket(text) -> Pocket:
    """parse_pocket (io.cpp:162-206); raises ParseError (RangeError included) with the reference's
    message."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    lib = _load()
    h = C.c_void_p()
    err = C.create_string_buffer(4096)
    rc = lib.gd_parse_pocket(data, len(data), C.byref(h), err, len(err))
    if rc:
        raise _ERRORS.get(rc, GeoDockError)(err.value.decode(errors="replace"))
    try:
        dims, origin = np.zeros(3, np.uint32), np.zeros(3)
        sp, fp = C.c_double(), C.POINTER(C.c_double)()
        lib.gd_pocketbuf_view(h, _p(dims, _u32p), _p(origin, _f64p), C.byref(sp), C.byref(fp))
        n = int(np.prod(dims.astype(np.uint64)))
        field = np.ctypeslib.as_array(fp, shape=(n,)).copy()
        return Pocket(tuple(int(x) for x in dims), tuple(float(x) for x in origin), float(sp.value), field)
    finally:
        lib.gd_pocketbuf_free(h)


def load_pocket(path: str) -> Pocket:
    """load_pocket (io.cpp:271-274)."""
    with open(path, "rb") as f:
        return parse_pocket(f.read())


def serialize_pocket(p: Pocket) -> str:
    """serialize_pocket (io.cpp:208-214): header lines, then 12 values per line."""
    out = [f"origin {format_double(p.origin[0])} {format_double(p.origin[1])} {format_double(p.origin[2])}\n",
           f"spacing {format_double(p.spacing)}\n", f"dims {p.dims[0]} {p.dims[1]} {p.dims[2]}\n"]
    f = np.asarray(p.field).ravel()
    for i, v in enumerate(f):
        out.append(format_double(v) + ("\n" if (i + 1) % 12 == 0 or i + 1 == len(f) else " "))
    return "".join(out)


def format_double(v: float) -> str:
    """format_double (io.cpp:14-18): %.9g."""
    return "%.9g" % v


def serialize_library(lib: Library) -> str:
    """serialize_ligand_library (io.cpp:143-160)."""
    out = []
    for i in range(lib.n_ligands):
        a0, a1 = int(lib.atom_off[i]), int(lib.atom_off[i + 1])
        b0, b1 = int(lib.bond_off[i]), int(lib.bond_off[i + 1])
        r0, r1 = int(lib.rot_off[i]), int(lib.rot_off[i + 1])
        out.append(f"ligand {lib.name(i)}\natoms {a1 - a0}\n")
        for a in range(a0, a1):
            x, y, z = lib.xyz[a]
            out.append(f"{format_double(x)} {format_double(y)} {format_double(z)} {format_double(lib.radius[a])}\n")
        out.append(f"bonds {b1 - b0}\n" + "".join(f"{int(p)} {int(q)}\n" for p, q in lib.bonds[b0:b1]))
        out.append(f"rotamers {r1 - r0}\n" + "".join(f"{int(p)} {int(q)}\n" for p, q in lib.rots[r0:r1]) + "end\n")
    return "".join(out)


def write_results(lib: Library, res: "DockResults") -> str:
    """write_results (io.cpp:216-223): the results CSV, one row per ligand in library order."""
    rows = ["ligand_name,best_score,best_restart_id,score_calls,align_seconds,optimize_seconds\n"]
    for i in range(lib.n_ligands):
        rows.append(f"{lib.name(i)},{format_double(res.best_score[i])},{int(res.best_restart[i])},"
                    f"{int(res.score_calls[i])},{format_double(res.phase_times[2 * i])},"
                    f"{format_double(res.phase_times[2 * i + 1])}\n")
    return "".join(rows)


def write_metrics(m: RunMetrics, config: NodeConfig) -> str:
    """write_metrics (io.cpp:225-245): the one-row run metrics CSV."""
    busy, idle, wait = sum(m.device_busy_seconds), sum(m.device_idle_seconds), sum(m.worker_wait_seconds)
    mean_wait = wait / m.ligand_count if m.ligand_count > 0 else 0.0
    return ("workers,devices,lane_width,mode,ligands,wall_seconds,throughput,"
            "device_busy_seconds,device_idle_seconds,mean_lane_wait_seconds,"
            "align_seconds_total,optimize_seconds_total,lane_failures,exclusivity_violations\n"
            f"{config.n_workers},{config.n_devices},{config.lane_width},"
            f"{'synthetic' if config.mode == 'synthetic' else 'real'},{m.ligand_count},"
            f"{format_double(m.wall_seconds)},{format_double(m.throughput)},{format_double(busy)},"
            f"{format_double(idle)},{format_double(mean_wait)},{format_double(m.align_seconds_total)},"
            f"{format_double(m.optimize_seconds_total)},{m.lane_failures},{m.exclusivity_violations}\n")


def moving_set(lib: Library, i: int, r: int) -> np.ndarray:
    """Rotamer r's moving set (finalize_ligand, molecule.cpp:88-98)."""
    L, keep = lib._c()
    out = np.zeros(max(1, lib.n_atoms(i)), np.uint32)
    n = C.c_uint32()
    rc = _load().gd_moving_set(C.byref(L), i, r, _p(out, _u32p), C.byref(n))
    if rc:
        raise _ERRORS.get(rc, GeoDockError)(f"gd_moving_set failed ({rc})")
    return out[:n.value].copy()


# ----------------------------------------------------------------------------- device context
class Context:
    """One GPU (gd_ctx). Externally synchronized, like the reference's DeviceLane guard."""

    def __init__(self, device: int = 0, mode: Optional[int] = None):
        self._lib = _load()
        h = C.c_void_p()
        rc = self._lib.gd_create(device, C.byref(h))
        if rc != GD_OK:
            raise DeviceError(f"gd_create(device={device}) failed with status {rc}; a CUDA device is required "
                              "(there is no CPU fallback)")
        self._h = h
        self.device = device
        # a context is externally synchronized (one batch in flight, like the reference's lane
        # guard, pipeline.cpp:75,138); run_screening threads sharing a device take this lock
        self.lock = threading.RLock()
        self.pocket = None
        self.params = DockParams()
        if mode is not None:
            self.set_mode(mode)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.gd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc):
        if rc != GD_OK:
            msg = self._lib.gd_last_error(self._h).decode(errors="replace")
            raise _ERRORS.get(rc, GeoDockError)(msg)

    @property
    def stream_ptr(self) -> int:
        return int(self._lib.gd_stream(self._h) or 0)

    def set_mode(self, mode: int):
        self._check(self._lib.gd_set_mode(self._h, mode))

    def set_pocket(self, pocket: Pocket):
        if pocket is self.pocket:
            return
        d = np.asarray(pocket.dims, np.uint32)
        o = np.asarray(pocket.origin, np.float64)
        f = np.ascontiguousarray(pocket.field, np.float64)
        if f.size and not (f.min() >= 0.0 and f.max() <= 1.0):
            warnings.warn("pocket field lies outside [0, 1] (the Pocket contract, scoring.hpp:15): "
                          "batches on this pocket run the all-FP64 kernel, not the fast path "
                          "(stats()['exact_fallback'] == 1)", RuntimeWarning, stacklevel=2)
        self._check(self._lib.gd_set_pocket(self._h, _p(d, _u32p), _p(o, _f64p), pocket.spacing, _p(f, _f64p)))
        self.pocket = pocket

    def set_params(self, params: DockParams):
        if params == self.params and getattr(self, "_params_set", False):
            return
        self._check(self._lib.gd_set_params(self._h, C.byref(params._c())))
        self.params = DockParams(**params.__dict__)
        self._params_set = True

    def _alloc_results(self, lib: Library, trace: bool):
        L, A, Rt = lib.n_ligands, int(lib.atom_off[-1]), int(lib.rot_off[-1])
        N, reps = self.params.n_restarts, self.params.num_repetitions
        # gd_dock_batch writes every element of these (a failed call raises), so they are not
        # zero-filled first: np.zeros of a heap-recycled 10 MB block is a memset (~1.5 ms per 10k)
        out = DockResults(np.empty(L), np.empty(L, np.uint32), np.empty(L, np.uint64), np.empty(2 * L),
                          np.empty((A, 3)), np.empty(Rt))
        if trace:
            out.align_index = np.zeros(L * N, np.uint32)
            out.align_score = np.zeros(L * N)
            out.restart_score = np.zeros(L * N)
            out.step_k = np.zeros(Rt * N * reps, np.int32)
        r = _Results()
        r.best_score, r.best_restart = _p(out.best_score, _f64p), _p(out.best_restart, _u32p)
        r.score_calls, r.phase_times = _p(out.score_calls, _u64p), _p(out.phase_times, _f64p)
        r.final_xyz, r.final_dihedrals = _p(out.final_xyz, _f64p), _p(out.final_dihedrals, _f64p)
        r.align_index, r.align_score = _p(out.align_index, _u32p), _p(out.align_score, _f64p)
        r.restart_score, r.step_k = _p(out.restart_score, _f64p), _p(out.step_k, _i32p)
        return out, r

    def dock(self, lib: Library, pocket: Pocket = None, params: DockParams = None, trace=False) -> DockResults:
        """gd_dock_batch: host arrays in, host arrays out (validate, pack, H2D, kernels, D2H)."""
        if pocket is not None:
            self.set_pocket(pocket)
        if params is not None:
            self.set_params(params)
        L, keep = lib._c()
        out, r = self._alloc_results(lib, trace)
        self._check(self._lib.gd_dock_batch(self._h, C.byref(L), C.byref(r)))
        return out

    def stage(self, lib: Library) -> "Batch":
        L, keep = lib._c()
        b = C.c_void_p()
        self._check(self._lib.gd_stage(self._h, C.byref(L), C.byref(b)))
        return Batch(self, b, lib)

    def stats(self) -> dict:
        s = _Stats()
        self._check(self._lib.gd_last_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def profile(self, lib: Library, pocket: Pocket = None, params: DockParams = None) -> dict:
        """The reference's `profile` subcommand (geodock_main.cpp:189-232) for the GPU path: the
        DockStats counters (docking.hpp:46-55, the closed forms the reference records: score calls
        N G + N reps R S, bump checks N reps R S, fragment rotations N reps R (S - 1)) and the
        align / optimize time split, here the device time of K1a (alignment) and K1b (exact
        refinement + dihedral sweep), plus the two-stage search's own counters."""
        if pocket is not None:
            self.set_pocket(pocket)
        if params is not None:
            self.set_params(params)
        p = self.params
        b = self.stage(lib)
        try:
            b.run()
            self.sync()
            ms = self.kernel_ms()
            st = self.stats()
        finally:
            b.free()
        N, reps, S = p.n_restarts, p.num_repetitions, p.dihedral_steps
        G = int(np.prod(p.rotation_steps))
        R = int(lib.rot_off[-1] - lib.rot_off[0]) if lib.n_ligands else 0
        t_a, t_o = ms["k1a_align"], ms["k1b_sweep"]
        tot = t_a + t_o
        return {"align_ligand": {"time_pct": 100.0 * t_a / tot if tot else 0.0, "visits": N * lib.n_ligands},
                "optimize_pose": {"time_pct": 100.0 * t_o / tot if tot else 0.0, "visits": N * reps * lib.n_ligands},
                "score_pose[align]": N * G * lib.n_ligands, "score_pose[optimize]": N * reps * R * S,
                "bump_check": N * reps * R * S, "rotate_fragment": N * reps * R * (S - 1),
                "total_score_calls": N * G * lib.n_ligands + N * reps * R * S,
                "expected_score_calls": sum(count_score_calls(p, int(lib.rot_off[i + 1] - lib.rot_off[i]))
                                            for i in range(lib.n_ligands)),
                "device_ms": ms, "kernel_stats": st}

    @staticmethod
    def format_profile(prof: dict) -> str:
        """The reference's profile table text (geodock_main.cpp:215-229)."""
        lines = ["function time_pct visits",
                 f"align_ligand {prof['align_ligand']['time_pct']:.2f} {prof['align_ligand']['visits']}",
                 f"optimize_pose {prof['optimize_pose']['time_pct']:.2f} {prof['optimize_pose']['visits']}"]
        for k in ("score_pose[align]", "score_pose[optimize]", "bump_check", "rotate_fragment",
                  "total_score_calls", "expected_score_calls"):
            lines.append(f"{k} - {prof[k]}")
        return "\n".join(lines) + "\n"

    def kernel_ms(self) -> dict:
        """Device time of the last gd_run's kernels (CUDA events on the context stream)."""
        ms = (C.c_float * 3)()
        self._check(self._lib.gd_last_kernel_ms(self._h, ms, 3))
        return {"k1a_align": ms[0], "k1b_sweep": ms[1], "k2_finalize": ms[2]}

    def run_times(self) -> dict:
        """Device accounting of the last dock() (gd_last_run_times), seconds."""
        t = (C.c_double * 4)()
        self._check(self._lib.gd_last_run_times(self._h, t, 4))
        return {"busy": t[0], "align": t[1], "optimize": t[2], "host_wait": t[3]}

    def sync(self):
        self._check(self._lib.gd_sync(self._h))


class Batch:
    """A staged, device-resident batch (gd_batch): run() enqueues kernels only."""

    def __init__(self, ctx: Context, handle, lib: Library):
        self.ctx, self._h, self.lib = ctx, handle, lib

    def run(self):
        self.ctx._check(self.ctx._lib.gd_run(self._h))

    def fetch(self, trace=False) -> DockResults:
        out, r = self.ctx._alloc_results(self.lib, trace)
        self.ctx._check(self.ctx._lib.gd_fetch(self._h, C.byref(r)))
        return out

    def topk_array(self, k: int) -> np.ndarray:
        """gd_topk (K3): the k best ligands of the batch as an (n, 3) float64 array (best score,
        ligand index within the batch, best restart), ordered by (score desc, index asc)."""
        hits = (_Hit * max(1, k))()
        n = C.c_uint32()
        self.ctx._check(self.ctx._lib.gd_topk(self._h, k, hits, C.byref(n)))
        rec = np.frombuffer(hits, dtype=np.dtype([("s", "<f8"), ("l", "<u4"), ("r", "<u4")]), count=n.value)
        return np.stack([rec["s"], rec["l"].astype(np.float64), rec["r"].astype(np.float64)], axis=1)

    def topk(self, k: int):
        return [(float(s), int(i), int(r)) for s, i, r in self.topk_array(k)]

    def free(self):
        if self._h:
            self.ctx._lib.gd_batch_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ----------------------------------------------------------------------------- reference-shaped API
_default_ctx = {}
_default_ctx_lock = threading.Lock()


def _ctx_for(device: int) -> Context:
    """The shared per-device context (created once, under a module lock)."""
    with _default_ctx_lock:
        c = _default_ctx.get(device)
        if c is None:
            c = _default_ctx[device] = Context(device)
        return c


def dock_ligand(ligand: Library, pocket: Pocket, params: DockParams = DockParams(), device: int = 0) -> DockResult:
    """dock_ligand (docking.hpp:140-141) for a one-ligand Library (see make_ligand).

    Thread-safe like the reference's pure function: the shared per-device context is externally
    synchronized, so the pocket/params upload and the batch run under its lock."""
    if ligand.n_ligands != 1:
        raise ContractError("dock_ligand takes exactly one ligand")
    ctx = _ctx_for(device)
    with ctx.lock:
        res = ctx.dock(ligand, pocket, params)
    return res.result(ligand, 0)


def run_screening(library: Library, pocket: Pocket, params: DockParams = DockParams(), n_devices: int = 1,
                  devices: Optional[Sequence[int]] = None, trace: bool = False):
    """run_screening (pipeline.hpp:85-89) on GPUs: contiguous library shards, one host thread per GPU.

    Results come back in library order and are bit-identical for every device count (each result is
    a pure function of (ligand, pocket, params)). Returns (DockResults, RunMetrics).
    """
    if library.n_ligands == 0:
        raise ContractError("ligand library is empty")  # pipeline.cpp:192
    devs = list(devices) if devices is not None else list(range(max(1, n_devices)))
    L = library.n_ligands
    bounds = [L * i // len(devs) for i in range(len(devs) + 1)]
    parts, errors = [None] * len(devs), [None] * len(devs)
    times = [{"busy": 0.0, "align": 0.0, "optimize": 0.0, "host_wait": 0.0} for _ in devs]

    # every lane's context exists before any docks: each sizes its host pool by the live contexts
    for i, d in enumerate(devs):
        if bounds[i + 1] > bounds[i]:
            _ctx_for(d)

    def work(i):
        try:
            shard = library.slice(bounds[i], bounds[i + 1])
            if shard.n_ligands:
                ctx = _ctx_for(devs[i])
                with ctx.lock:
                    parts[i] = ctx.dock(shard, pocket, params, trace=trace)
                    times[i] = ctx.run_times()
        except BaseException as e:  # rethrown after join, like pipeline.cpp:262-272
            errors[i] = e

    t0 = time.perf_counter()
    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(devs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    wall = time.perf_counter() - t0
    for e in errors:
        if e is not None:
            raise e
    got = [p for p in parts if p is not None]
    cat = lambda k: None if getattr(got[0], k) is None else np.concatenate([getattr(p, k) for p in got])
    res = DockResults(**{k: cat(k) for k in DockResults.__dataclass_fields__})
    busy = [t["busy"] for t in times]
    m = RunMetrics(wall, L / wall if wall > 0 else 0.0, L, busy, [wall - b for b in busy],
                   [t["host_wait"] for t in times], sum(t["align"] for t in times),
                   sum(t["optimize"] for t in times))
    return res, m
