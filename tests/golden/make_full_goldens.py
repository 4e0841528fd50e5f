"""Full-library goldens from the UNMODIFIED reference (the libraries bench.py times).

Run here (needs /root/reference and `make -C oracle ref`; ~15 CPU-minutes on 8 cores):
    python tests/golden/make_full_goldens.py
For each case the reference's own run_screening (pipeline.cpp:187-290, n_devices = 0, all host
threads) docks the whole library; best_score (FP64 bits) and best_restart of every ligand are
stored (`full_<case>.npz`) with their sha256 digest. tests/test_gpu_full.py reproduces them on the
GPU bit for bit. Nothing on the GPU box reads /root/reference.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from oracle import Oracle, Params  # noqa: E402

CASES = {
    # name: (count, atoms, rotamers, pocket kwargs, params)
    "c2_default": (10000, 40, 8, {}, Params()),
    "c2_clash01": (10000, 40, 8, {}, Params(clash_factor=0.1)),
    "c4_clash01": (1000, 120, 32, {}, Params(clash_factor=0.1)),
    "c5s_default": (10000, 40, 8, dict(dims=(47, 47, 47), spacing=0.375), Params()),
}


def digest(best, rid):
    return hashlib.sha256(np.ascontiguousarray(best, "<f8").tobytes() +
                          np.ascontiguousarray(rid, "<u4").tobytes()).hexdigest()


def main(names):
    ref = Oracle("reference")
    nproc = len(os.sched_getaffinity(0))
    for name in names:
        count, atoms, rots, pk, params = CASES[name]
        pocket = ref.make_pocket(**pk)
        lib = ref.make_library(count, atoms, rots, 0)
        t = time.time()
        best, rid, wall = ref.run_screening(lib, pocket, params, n_workers=nproc)
        d = digest(best, rid)
        np.savez_compressed(os.path.join(HERE, f"full_{name}.npz"), best_score=best, best_restart=rid,
                            sha256=d, spec=json.dumps(dict(count=count, atoms=atoms, rotamers=rots, pocket=pk,
                                                           params=params.__dict__)))
        print(name, d[:16], f"{count / wall:.1f} lig/s ({nproc} threads, {time.time() - t:.0f} s)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
