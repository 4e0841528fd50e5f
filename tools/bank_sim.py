"""Shared-memory wavefront model of K1a's cell gathers (LDS.128: 4 phases of 8 lanes; a phase costs
the largest number of distinct 16-byte cells that fall into one of the 8 bank quads). Explores
lane -> work mappings and cell layouts on the C2 library with uniform random start poses.

usage: python tools/bank_sim.py [ligands]
"""
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1901_06229_b200 as gd  # noqa: E402

rng = np.random.default_rng(1)
L = int(sys.argv[1]) if len(sys.argv) > 1 else 20
lib = gd.make_library(gd.LibrarySpec(L, 40, 8, 0))
pk = gd.make_pocket()
dims = np.array(pk.dims)
cdim = dims - 1
sp = pk.spacing
org = np.array(pk.origin)
lo, hi = np.array(pk.bounds_lo()), np.array(pk.bounds_hi())


def rz(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]])


def ry(b):
    c, s = np.cos(b), np.sin(b)
    return np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]])


na, nb, nc = 16, 16, 8
frames = [(j, k) for j in range(nb) for k in range(nc)]
F = {f: ry(np.pi * f[0] / (nb - 1)) @ rz(2 * np.pi * f[1] / nc) for f in frames}
kept = [f for f in frames if not (f[0] in (0, nb - 1) and f[1] > 0)]
nq = na // 4
units = [(f, c0) for f in kept for c0 in (0, 2)]


def rand_rot():
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def cells_for(atoms, t, lane_units):
    """cell index [lane, atom, gi, q] (dummy = -1) for 32 lanes' units"""
    out = np.full((32, len(atoms), 2, 4), -1, np.int64)
    for l, u in enumerate(lane_units):
        if u is None:
            continue
        f, c0 = u
        for gi in range(2):
            for q in range(4):
                ia = c0 + gi + q * nq
                R = rz(2 * np.pi * ia / na) @ F[f]
                g = (atoms @ R.T + t - org) / sp
                inside = np.all((g >= 0) & (g < cdim), axis=1)
                ijk = np.floor(g).astype(np.int64)
                idx = np.where(inside, ijk[:, 0] + cdim[0] * ijk[:, 1] + cdim[0] * cdim[1] * ijk[:, 2], -1)
                out[l, :, gi, q] = idx
    return out


def wavefronts(addr, color):
    """addr [32] cell indices (-1 dummy) -> wavefronts of one LDS.128 under the 4x8 phase model"""
    tot = 0
    for ph in range(4):
        a = addr[8 * ph:8 * ph + 8]
        a = np.unique(a)
        cols = color(a)
        tot += np.bincount(cols, minlength=8).max()
    return tot


def run(mapping, color, restarts=2):
    wf = n = 0
    for li in range(L):
        xyz = lib.xyz[lib.atom_off[li]:lib.atom_off[li + 1]]
        for _ in range(restarts):
            R0 = rand_rot()
            atoms = (xyz - xyz.mean(0)) @ R0.T
            t = rng.uniform(lo, hi)
            for mu_units in mapping():
                c = cells_for(atoms, t, mu_units)
                for a in range(len(atoms)):
                    for gi in range(2):
                        for q in range(4):
                            wf += wavefronts(c[:, a, gi, q], color)
                            n += 1
    return wf / n


def map_current():
    for mu in range(7):
        yield [units[l + 32 * mu] for l in range(32)]


cx, cxy = cdim[0], cdim[0] * cdim[1]
layouts = {
    "linear x-fastest (current)": lambda a: np.where(a < 0, 0, a) % 8,
}
if __name__ == "__main__":
    for name, col in layouts.items():
        print(f"{name:32s} current mapping: {run(map_current, col):.3f} wavefronts / LDS.128")


def ijk(a):
    a = np.where(a < 0, 0, a)
    return a % cx, (a // cx) % cdim[1], a // cxy


layouts["parity (x&1)+2(y&1)+4(z&1)"] = lambda a: (lambda i, j, k: (i & 1) + 2 * (j & 1) + 4 * (k & 1))(*ijk(a))
layouts["x+2y+4z"] = lambda a: (lambda i, j, k: (i + 2 * j + 4 * k) % 8)(*ijk(a))
layouts["x+3y+5z"] = lambda a: (lambda i, j, k: (i + 3 * j + 5 * k) % 8)(*ijk(a))
layouts["x+2y+3z"] = lambda a: (lambda i, j, k: (i + 2 * j + 3 * k) % 8)(*ijk(a))
layouts["random hash"] = lambda a: (np.where(a < 0, 0, a) * 2654435761 >> 7) % 8


def map_meridian():
    """quarter-warp = 8 consecutive beta rows at one (gamma, c0); rows 0 and 15 hold 1 kept frame each"""
    order = []
    by = {}
    for (f, c0) in units:
        by.setdefault((f[1], c0), []).append((f, c0))
    for key in sorted(by):
        order += sorted(by[key], key=lambda u: u[0][0])
    for mu in range(7):
        yield [order[l + 32 * mu] for l in range(32)]


def map_gamma():
    """quarter-warp = the 8 gammas of one beta row (same c0)"""
    order = sorted(units, key=lambda u: (u[0][0], u[1], u[0][1]))
    for mu in range(7):
        yield [order[l + 32 * mu] for l in range(32)]


if __name__ == "__main__":
    for mname, m in (("meridian", map_meridian), ("gamma", map_gamma)):
        for name, col in layouts.items():
            print(f"{name:32s} {mname} mapping: {run(m, col):.3f}")
