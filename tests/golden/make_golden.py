"""Generates the committed golden vectors in tests/golden/ from the UNMODIFIED reference.

Run here (needs /root/reference and `make -C oracle ref`):  python tests/golden/make_golden.py
The outputs are small .npz files; tests compare the oracle restatement and the GPU path to them
bit-for-bit. Nothing at run time on the GPU box reads /root/reference.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from oracle import Oracle, Params, SplitMix64, random_ligand_spec, random_pocket_spec  # noqa: E402

ref = Oracle("reference")


def dock_case(name, count, atoms, rotamers, params, lib_seed=0, pocket_kw=None):
    pocket = ref.make_pocket(**(pocket_kw or {}))
    lib = ref.make_library(count, atoms, rotamers, lib_seed)
    out = ref.dock(lib, pocket, params, trace=True)
    np.savez_compressed(os.path.join(HERE, name + ".npz"),
                        spec=json.dumps(dict(count=count, atoms=atoms, rotamers=rotamers, lib_seed=lib_seed,
                                             pocket=pocket_kw or {}, params=params.__dict__)),
                        best_score=out.best_score, best_restart=out.best_restart, score_calls=out.score_calls,
                        phase=out.phase, final_xyz=out.final_xyz, final_dih=out.final_dih,
                        align_index=out.align_index, align_score=out.align_score,
                        restart_score=out.restart_score, step_k=out.step_k, step_score=out.step_score)
    print(name, "mean best", out.best_score.mean(), "commits", int((out.step_k > 0).sum()))


def random_instances(name, n, seed, clash):
    """acceptance #2 (acceptance_main.cpp:100-165): random pocket + ligand + params per instance."""
    rng = SplitMix64(seed)
    rows = []
    for i in range(n):
        pk = random_pocket_spec(rng)
        lk = random_ligand_spec(rng, 10, 3)
        params = Params(n_restarts=1 + rng.below(4), rotation_steps=(6, 6, 4),
                        num_repetitions=1 + rng.below(2), dihedral_steps=4 + rng.below(7),
                        clash_factor=clash, seed=rng.next())
        pocket = ref.make_pocket(**pk)
        lib = ref.make_library(**lk)
        out = ref.dock(lib, pocket, params, trace=True)
        rows.append(dict(pocket=pk, ligand=lk, params=params.__dict__, best_score=float(out.best_score[0]).hex(),
                         best_restart=int(out.best_restart[0]), score_calls=int(out.score_calls[0]),
                         final_xyz=[float(x).hex() for x in out.final_xyz.ravel()],
                         final_dih=[float(x).hex() for x in out.final_dih],
                         align_index=out.align_index.tolist(), step_k=out.step_k.tolist()))
    with open(os.path.join(HERE, name + ".json"), "w") as f:
        json.dump(rows, f)
    print(name, len(rows))


def unit_pins():
    pocket = ref.make_pocket()
    rng = np.random.default_rng(0)
    pts = rng.uniform(-1.0, 18.5, size=(2000, 3))
    # exact faces / corners / nodes (scoring_test.cpp:30-59 style)
    extra = np.array([[0, 0, 0], [17.25, 17.25, 17.25], [17.25, 3.0, 3.0], [0.75, 1.5, 2.25],
                      [-1e-12, 3, 3], [17.25 + 1e-12, 3, 3], [3.0, 3.0, 17.25 - 1e-13]], float)
    pts = np.vstack([pts, extra])
    vals = ref.sample_field(pocket, pts)
    grid = ref.rotation_grid((16, 16, 8))
    np.savez_compressed(os.path.join(HERE, "unit_pins.npz"), pts=pts, sample=vals, grid=grid,
                        grid_small=ref.rotation_grid((6, 5, 4)),
                        pocket_sha256=hashlib.sha256(pocket.field.tobytes()).hexdigest(),
                        fine_sha256=hashlib.sha256(ref.make_pocket(dims=(47, 47, 47), spacing=0.375).field.tobytes()).hexdigest(),
                        lib_c2_sha256=hashlib.sha256(b"".join(getattr(ref.make_library(64, 40, 8, 0), k).tobytes()
                                                              for k in ("xyz", "radius", "bonds", "rots"))).hexdigest())
    print("unit pins", len(pts))


if __name__ == "__main__":
    unit_pins()
    if sys.argv[1:] == ["pins"]:
        sys.exit(0)
    dock_case("c1_default", 100, 32, 4, Params())
    dock_case("c1_clash01", 100, 32, 4, Params(clash_factor=0.1))
    dock_case("c2_prefix_default", 24, 40, 8, Params())
    dock_case("c2_prefix_clash01", 24, 40, 8, Params(clash_factor=0.1))
    dock_case("c4_prefix_clash01", 4, 120, 32, Params(clash_factor=0.1))
    dock_case("c5_prefix_default", 8, 40, 8, Params(), pocket_kw=dict(dims=(47, 47, 47), spacing=0.375))
    random_instances("random_clash075", 100, 20250807, 0.75)
    random_instances("random_clash03", 100, 777, 0.3)
