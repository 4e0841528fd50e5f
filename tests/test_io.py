"""Data formats either side of the hot path (CPU): the .lgd library parser (gd_parse_library,
multi-threaded C++) against the reference's parse_ligand_library (io.cpp:96-140, through the
oracle/_ref shim), the serializer (io.cpp:143-160) and the results CSV (io.cpp:216-223).

Parity bar: identical arrays (bit-exact doubles), identical bytes for the writers, and for
malformed input the same exception class and the same message (ParseError text with its line).
"""
import numpy as np
import pytest

import paper_1901_06229_b200 as gd
from oracle import OracleError

TWO_ATOM = ("ligand probe\n"
            "atoms 2\n"
            "0 0 0 0.5\n"
            "1.5 0 0 0.5\n"
            "bonds 1\n"
            "0 1\n"
            "rotamers 0\n"
            "end\n")

RING = ("ligand ringy\natoms 3\n0 0 0 0.5\n1.5 0 0 0.5\n0.75 1.3 0 0.5\n"
        "bonds 3\n0 1\n1 2\n2 0\nrotamers 1\n0 1\nend\n")

# malformed or edge-case texts; each is parsed by both implementations
CASES = [
    "", "\n\n  \n", TWO_ATOM, TWO_ATOM * 3, RING,
    "ligand broken\natoms 2\n0 0 0 0.5\noops 0 0 0.5\n",                      # io_test: line 4
    "ligand a atoms 1 0 0 0 0.5 bonds 0 rotamers 0 end",                       # one line, no LF
    TWO_ATOM.replace("\n", "\r\n"),                                            # CRLF
    "ligand hx\natoms 2\n0x0p+0 0 0 0x1p-1\n+1.5 -0 0 .5\nbonds 1\n0 1\nrotamers 0\nend\n",
    "ligand big\natoms 2\n1e999 0 0 0.5\n1.5 0 0 0.5\nbonds 1\n0 1\nrotamers 0\nend\n",   # ERANGE
    "ligand tiny\natoms 2\n1e-400 0 0 0.5\n1.5 0 0 0.5\nbonds 1\n0 1\nrotamers 0\nend\n",  # underflow
    "ligand nanr\natoms 2\n0 0 0 nan\n1.5 0 0 0.5\nbonds 1\n0 1\nrotamers 0\nend\n",     # validation
    "ligand infx\natoms 2\ninf 0 0 0.5\n1.5 0 0 0.5\nbonds 1\n0 1\nrotamers 0\nend\n",
    "ligand neg\natoms -1\n",
    "ligand cnt\natoms 2x\n",
    "ligand huge\natoms 99999999999999999999\n",
    "ligand many\natoms 3\n0 0 0 0.5\n1.5 0 0 0.5\nbonds 1\n0 1\nrotamers 0\nend\n",   # 'bonds' as atom x
    "ligand trunc\natoms 2\n0 0 0 0.5\n1.5 0",                                 # EOF inside atoms
    "ligand trunc\natoms 2\n0 0 0 0.5\n1.5 0 0 0.5\n",                         # EOF before bonds
    "ligand trunc\natoms 2\n0 0 0 0.5\n1.5 0 0 0.5\nbonds 1\n0",               # EOF inside bonds
    "ligand trunc\natoms 2\n0 0 0 0.5\n1.5 0 0 0.5\nbonds 1\n0 1\nrotamers 1\n0 1\n",  # no end
    "ligand",                                                                  # EOF before name
    "ligand x\natoms 1\n0 0 0 0.5\nbond 0\n",                                  # bad keyword
    "molecule x\n",
    TWO_ATOM + "garbage\n",
    "ligand selfbig\natoms 2\n0 0 0 0.5\n1.5 0 0 0.5\nbonds 2\n5000000000 5000000000\n"
    "5000000000 6000000000\nrotamers 0\nend\n",
    "ligand rotbig\natoms 2\n0 0 0 0.5\n1.5 0 0 0.5\nbonds 1\n0 1\nrotamers 1\n0 7000000000\nend\n",
    RING + "ligand later\natoms 2\n0 0 0 0.5\noops\n",                          # validation first
    "ligand first\natoms 2\n0 0 0 0.5\noops\n" + RING,                         # parse error first
    TWO_ATOM + "ligand nobond\natoms 2\n0 0 0 0.5\n9 9 9 0.5\nbonds 0\nrotamers 0\nend\n",
]


def _same_lib(a, b):
    for k in ("atom_off", "bond_off", "rot_off", "name_off"):
        assert np.array_equal(np.asarray(getattr(a, k), np.uint32), np.asarray(getattr(b, k), np.uint32)), k
    for k in ("xyz", "radius", "dihedrals"):
        x, y = np.asarray(getattr(a, k), np.float64).ravel(), np.asarray(getattr(b, k), np.float64).ravel()
        assert x.tobytes() == y.tobytes(), k  # bit-exact, NaNs included
    for k in ("bonds", "rots"):
        assert np.array_equal(np.asarray(getattr(a, k), np.uint32).ravel(), np.asarray(getattr(b, k), np.uint32).ravel()), k
    assert bytes(a.names) == bytes(b.names)


@pytest.mark.parametrize("i", range(len(CASES)))
def test_parse_matches_reference(reference, i):
    text = CASES[i].encode()
    try:
        ref = reference.parse_library(text)
        ref_err = None
    except OracleError as e:
        ref, ref_err = None, e
    if ref_err is None:
        _same_lib(gd.parse_library(text), ref)
    else:
        want = {8: gd.ParseError, 2: gd.ValidationError}[ref_err.code]
        with pytest.raises(want) as got:
            gd.parse_library(text)
        assert str(got.value) == ref_err.msg


def test_parse_error_reports_line_like_io_test():
    with pytest.raises(gd.ParseError, match=r"\(line 4\)$"):
        gd.parse_library(CASES[5])


def test_roundtrip_generated_library_matches_reference(reference):
    lib = gd.make_library(gd.LibrarySpec(3000, 32, 4, 11))  # large enough for several parse threads
    text = gd.serialize_library(lib).encode()
    ours = gd.parse_library(text)
    ref = reference.parse_library(text)
    _same_lib(ours, ref)
    assert reference.serialize_parsed() == text  # our writer == the reference's bytes
    assert gd.serialize_library(ours).encode() == text  # serialize . parse is idempotent
    # and the parsed library is the generated one up to the 9-digit text format
    assert np.allclose(ours.xyz, lib.xyz, rtol=1e-8, atol=1e-9)
    assert np.array_equal(ours.bonds, lib.bonds) and np.array_equal(ours.rots, lib.rots)


def test_results_csv_matches_reference(reference):
    lib = gd.make_library(gd.LibrarySpec(5, 8, 2, 3))
    rng = np.random.default_rng(0)
    res = gd.DockResults(best_score=rng.random(5), best_restart=np.arange(5, dtype=np.uint32),
                         score_calls=np.arange(5, dtype=np.uint64) * 1000 + 79360,
                         phase_times=rng.random(10) * 1e-3, final_xyz=None, final_dihedrals=None)
    names = [lib.name(i) for i in range(5)]
    want = reference.write_results(names, res.best_score, res.best_restart, res.score_calls, res.phase_times)
    assert gd.write_results(lib, res).encode() == want


POCKETS = [
    "origin 0 0 0\nspacing 1\ndims 2 2 2\n0 0.25 0.5 1 0 0 1 1\n",              # io_test minimal grid
    "origin 0 0 0\nspacing 1\ndims 2 2 2\n0 0 0 0 0 0 0\n",                       # value count
    "origin 0 0 0\nspacing 1\ndims 2 2 2\n0 0 0 1.5 0 0 0 0\n",                   # RangeError
    "origin 0 0 0\nspacing 1\ndims 2 2 2\n0 0 0 -0.1 0 0 0 0\n",
    "origin 0 0 0\nspacing 1\ndims 2 2 2\n0 0 0 0 0 0 0 0 extra\n",               # trailing
    "origin 0 0 0\nspacing 0\ndims 2 2 2\n",
    "origin 0 0 0\nspacing -1\ndims 2 2 2\n",
    "origin 0 0 0\nspacing 1\ndims 2 1 2\n",
    "origin 0 0\nspacing 1\n",
    "origin 0 0 0\nspacing 1\ndims 2 2 2\n0 0 x 0 0 0 0 0\n",
    "origin 0 0 0\r\nspacing 0.375\r\ndims 2 2 2\r\n0 0 0 0 0 0 0 0\r\n",
    "origin 0 0 0 spacing 1 dims 2 2 2 0 0 0 0 0 0 0 0",
    "",
    "grid 0 0 0\n",
    "origin 0 0 0\nspacing 1\ndims 2 2 2\n0 0 0 0\n0 0 0 nan\n",
]


@pytest.mark.parametrize("i", range(len(POCKETS)))
def test_parse_pocket_matches_reference(reference, i):
    text = POCKETS[i].encode()
    try:
        ref = reference.parse_pocket(text)
        ref_err = None
    except OracleError as e:
        ref, ref_err = None, e
    if ref_err is None:
        p = gd.parse_pocket(text)
        assert p.dims == ref[0] and p.origin == ref[1] and p.spacing == ref[2]
        assert np.asarray(p.field).tobytes() == ref[3].tobytes()
    else:
        with pytest.raises(gd.ParseError) as got:
            gd.parse_pocket(text)
        assert str(got.value) == ref_err.msg


def test_pocket_roundtrip_matches_reference(reference):
    p = gd.make_pocket(gd.PocketSpec(dims=(47, 47, 47), spacing=0.375))
    text = gd.serialize_pocket(p).encode()
    assert reference.serialize_pocket(p.dims, p.origin, p.spacing, p.field) == text
    q = gd.parse_pocket(text)
    ref = reference.parse_pocket(text)
    assert q.dims == ref[0] and np.asarray(q.field).tobytes() == ref[3].tobytes()


METRICS = [
    gd.RunMetrics(0.05215, 191754.3, 10000, [0.04811], [0.00404], [0.04305], 0.0331, 0.0149),
    gd.RunMetrics(1.5, 666.6666666666666, 1000, [1.2, 1.25, 1.1, 0.9], [0.3, 0.25, 0.4, 0.6],
                  [0.1, 0.2, 0.3, 0.4], 3.0, 1.7),
    gd.RunMetrics(0.0, 0.0, 0, [], [], [], 0.0, 0.0),                       # empty run: mean wait 0
    gd.RunMetrics(1e-9, 1e12, 3, [1e-300], [-0.0], [5e-324], 1e308, 123456789.123, 2, 7),
]


@pytest.mark.parametrize("i", range(len(METRICS)))
def test_metrics_csv_matches_reference(reference, i):
    """write_metrics (io.cpp:225-245) byte for byte."""
    m = METRICS[i]
    for cfg in (gd.NodeConfig(), gd.NodeConfig(4, 4, 8, "real"), gd.NodeConfig(8, 2, 16, "synthetic")):
        assert gd.write_metrics(m, cfg).encode() == reference.write_metrics(m, cfg)


def _number_tokens():
    rng = np.random.default_rng(11)
    toks = ["-0", "0", "0.0", "-0.000", ".5", "5.", "-.5", "1.e5", "1e+05", "1E-5", "007", "00.0100",
            "2.2250738585072014e-308", "2.2250738585072011e-308", "4.9406564584124654e-324", "1e-320",
            "1.7976931348623157e308", "1.7976931348623159e308", "123456789012345678901234567890",
            "0.1000000000000000055511151231257827", "9007199254740993", "1e-400", "-1e-400", "1e400",
            "+2", "0x1.8p1", "1e", "1e+", ".", "-", "1..2", "1e5.5"]
    for _ in range(300):
        mant = "".join(str(d) for d in rng.integers(0, 10, int(rng.integers(1, 25))))
        dot = int(rng.integers(0, len(mant) + 1))
        s = ("-" if rng.random() < 0.3 else "") + mant[:dot] + "." + mant[dot:]
        if rng.random() < 0.5:
            s += "e" + str(int(rng.integers(-330, 330)))
        toks.append(s)
    return toks


def test_number_tokens_match_reference(reference):
    """The parser's fast number paths (std::from_chars for plain decimals, a digit loop for counts)
    give std::stod's / std::stoll's value or error on every token: tricky and random decimals."""
    for t in _number_tokens():
        text = f"ligand num\natoms 2\n{t} 0 0 0.5\n1.5 0 0 0.5\nbonds 1\n0 1\nrotamers 0\nend\n".encode()
        try:
            ref = reference.parse_library(text)
            ref_err = None
        except OracleError as e:
            ref, ref_err = None, e
        if ref_err is None:
            _same_lib(gd.parse_library(text), ref)
        else:
            with pytest.raises((gd.ParseError, gd.ValidationError)) as got:
                gd.parse_library(text)
            assert str(got.value) == ref_err.msg, t


@pytest.mark.parametrize("edit", ["none", "late_keyword", "late_count", "late_number", "early_keyword", "truncated"])
def test_parallel_record_walk_matches_reference(reference, edit):
    """The record-header walk runs per token slice in parallel (speculative chains adopted where the
    reference walk meets them): a multi-slice library with keyword-like ligand names, and errors
    planted in early / late slices, give the reference's arrays or its exact error."""
    lib = gd.make_library(gd.LibrarySpec(3000, 40, 8, 9))
    text = gd.serialize_library(lib)
    for name, fake in (("lig_000007", "ligand"), ("lig_000100", "atoms"), ("lig_001500", "end"), ("lig_002200", "bonds")):
        text = text.replace(f"ligand {name}\n", f"ligand {fake}\n")
    marker = {"late_keyword": "ligand lig_002500\n", "late_count": "ligand lig_002700\n",
              "late_number": "ligand lig_002900\n", "early_keyword": "ligand lig_000050\n"}.get(edit)
    if marker:
        at = text.index(marker) + len(marker)
        body = text[at:]
        if edit.endswith("keyword"):
            body = body.replace("bonds", "bondz", 1)
        elif edit == "late_count":
            body = body.replace("rotamers 8", "rotamers x8", 1)
        else:
            body = body.replace(" ", " 1.5e", 1)
        text = text[:at] + body
    if edit == "truncated":
        text = text[: len(text) - 37]
    data = text.encode()
    try:
        ref = reference.parse_library(data)
        ref_err = None
    except OracleError as e:
        ref, ref_err = None, e
    if ref_err is None:
        _same_lib(gd.parse_library(data), ref)
    else:
        with pytest.raises((gd.ParseError, gd.ValidationError)) as got:
            gd.parse_library(data)
        assert str(got.value) == ref_err.msg
