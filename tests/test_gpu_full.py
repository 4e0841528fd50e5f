"""GPU parity on the libraries the benchmark times (full sizes, not prefixes).

* The unmodified reference's run_screening (oracle/_ref, run here by
  tests/golden/make_full_goldens.py) docked the full C2 library (10k ligands) at the default clash
  0.75 and at clash 0.1, the full C4 library (1k x 120 atoms x 32 rotamers) at clash 0.1 and the
  10k C5-grid library; the GPU must reproduce every ligand's best score (FP64 bits) and best restart,
  i.e. the committed sha256 digests (the reference bar: dock_ligand bit for bit against the oracle,
  docking_test.cpp:322-338, and acceptance #2, acceptance_main.cpp:100-165).
* The fast two-stage kernels equal the all-FP64 kernel on every output and decision-trace bit of
  the same full libraries.
* A 20k random sample of the 1M-ligand C5 stream (the north star's screening sweep): the fast
  path over the whole million through the executor equals the FP64 kernel on the sample.
"""
import hashlib

import numpy as np
import pytest

import paper_1901_06229_b200 as gd
from conftest import load_npz

pytestmark = pytest.mark.gpu

FIELDS = ("best_score", "best_restart", "final_xyz", "final_dihedrals", "align_index", "align_score",
          "restart_score", "step_k", "score_calls")


def digest(best, rid):
    return hashlib.sha256(np.ascontiguousarray(best, "<f8").tobytes() +
                          np.ascontiguousarray(rid, "<u4").tobytes()).hexdigest()


def case(name):
    d = load_npz("full_" + name)
    sp = d["spec"]
    pocket = gd.make_pocket(gd.PocketSpec(**{k: tuple(v) if isinstance(v, list) else v
                                              for k, v in sp["pocket"].items()}))
    lib = gd.make_library(gd.LibrarySpec(sp["count"], sp["atoms"], sp["rotamers"], 0))
    params = gd.DockParams(**{k: tuple(v) if isinstance(v, list) else v for k, v in sp["params"].items()})
    return d, pocket, lib, params


@pytest.fixture(scope="module")
def pair():
    fast, exact = gd.Context(0, mode=gd.MODE_FAST), gd.Context(0, mode=gd.MODE_EXACT)
    yield fast, exact
    fast.close()
    exact.close()


def _first_diff(a, b):
    bad = np.flatnonzero(a != b)
    return None if bad.size == 0 else int(bad[0])


@pytest.mark.parametrize("name", ["c2_default", "c2_clash01", "c4_clash01", "c5s_default"])
def test_full_library_matches_reference_digest(pair, name):
    fast, exact = pair
    d, pocket, lib, params = case(name)
    out = fast.dock(lib, pocket, params, trace=True)
    i = _first_diff(out.best_score.view(np.uint64), d["best_score"].view(np.uint64))
    j = _first_diff(out.best_restart, d["best_restart"])
    assert i is None and j is None, f"{name}: first best_score mismatch at ligand {i}, best_restart at {j}"
    assert digest(out.best_score, out.best_restart) == str(d["sha256"])
    # the fast kernels against the all-FP64 kernel: every output and trace bit
    ref = exact.dock(lib, pocket, params, trace=True)
    for k in FIELDS:
        assert np.array_equal(getattr(out, k), getattr(ref, k)), (name, k)


def test_c5_million_stream_sample(pair):
    """The 1M-ligand C5 screen through the executor (gd_dock_batch, chunked and pipelined) on the fine
    47^3 grid; a seeded 20k random sample re-docked by the FP64 kernel equals it bit for bit."""
    fast, exact = pair
    pocket = gd.make_pocket(gd.PocketSpec(dims=(47, 47, 47), spacing=0.375))
    lib = gd.make_library(gd.LibrarySpec(1_000_000, 40, 8, 0))
    params = gd.DockParams()
    out = fast.dock(lib, pocket, params)
    idx = np.sort(np.random.default_rng(20251017).choice(lib.n_ligands, 20_000, replace=False))
    sub = lib.take(idx)
    ref = exact.dock(sub, pocket, params)
    assert np.array_equal(out.best_score[idx].view(np.uint64), ref.best_score.view(np.uint64))
    assert np.array_equal(out.best_restart[idx], ref.best_restart)
    rows = np.concatenate([np.arange(lib.atom_off[i], lib.atom_off[i + 1]) for i in idx])
    assert np.array_equal(out.final_xyz[rows], ref.final_xyz)
