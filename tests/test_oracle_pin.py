"""Pin the CPU restatement (oracle/plmss_oracle.c) before trusting it:
(1) the reference test-suite's own golden vectors (Fig. 1 fixture, code KATs,
per-code counts), (2) the golden fixtures produced by the reference library
(tests/golden/case_*.npz), (3) the compiled reference itself on fresh random
and tie-heavy grids (when oracle/_ref is present). CPU only."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, load_case


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- Fig. 1 --
@pytest.fixture(scope="module")
def fig1():
    return json.load(open(os.path.join(GOLDEN, "fig1.json")))


def test_fig1_labels_and_extrema(restatement, fig1):
    # proj/tests/test_segmentation.cpp:89-100, acceptance.cpp:67-92
    vals = np.array(fig1["order"])
    s = restatement.segment(fig1["dims"], values=vals)
    assert s["desc"].tolist() == fig1["desc"]
    assert s["asc"].tolist() == fig1["asc"]
    assert s["minima"].tolist() == [3, 12]
    assert s["maxima"].tolist() == [0, 15]
    rank = restatement.compute_order(vals)
    assert rank[s["minima"]].tolist() == [0, 1] and rank[s["maxima"]].tolist() == [14, 15]


def test_fig1_ms_regions(restatement, fig1):
    # proj/tests/test_segmentation.cpp:164-180
    s = restatement.segment(fig1["dims"], values=np.array(fig1["order"]))
    ms, keys = restatement.combine_ms(s["asc"], s["desc"])
    assert len(keys) == 4
    assert sorted(map(tuple, keys.tolist())) == [(3, 0), (3, 15), (12, 0), (12, 15)]
    for v in range(16):
        assert tuple(keys[ms[v]]) == (s["asc"][v], s["desc"][v])


def _segments(mesh):
    pts = mesh["points"][:, :2]
    out = []
    for p in range(len(mesh["source_cells"])):
        a, b = pts[2 * p].tolist(), pts[2 * p + 1].tolist()
        out.append(tuple(sorted([tuple(a), tuple(b)])))
    return sorted(out)


def _expected(segs):
    return sorted(tuple(sorted([(s[0], s[1]), (s[2], s[3])])) for s in segs)


def test_fig1_separator_networks(restatement, fig1):
    # proj/tests/test_marching.cpp:323-354
    s = restatement.segment(fig1["dims"], values=np.array(fig1["order"]))
    desc = restatement.emit_separators(fig1["dims"], s["desc"])
    assert _segments(desc) == _expected(fig1["desc_separators"])
    ms, _ = restatement.combine_ms(s["asc"], s["desc"])
    net = restatement.emit_separators(fig1["dims"], ms)
    assert _segments(net) == _expected(fig1["ms_separators"])


def test_fig1_boundaries(restatement, fig1):
    # proj/tests/test_marching.cpp:388-424
    s = restatement.segment(fig1["dims"], values=np.array(fig1["order"]))
    b = restatement.emit_boundaries(fig1["dims"], s["asc"])
    got = sorted((int(u), int(v), int(t)) for (u, v), t in zip(b["faces"], b["regions"][:, 0]))
    assert got == sorted(tuple(e) for e in fig1["asc_boundaries"])
    only3 = restatement.emit_boundaries(fig1["dims"], s["asc"], region_filter=3)
    assert len(only3["source_cells"]) == 3 and set(only3["regions"][:, 0].tolist()) == {3}


# ------------------------------------------------------------ code KATs --
KATS = [((7, 7, 9, 9), 10), ((7, 9, 9, 9), 21), ((1, 2, 3, 4), 27), ((5, 5, 5, 5), 0), ((5, 5, 5, 9), 3),
        ((5, 5, 9, 5), 8), ((5, 9, 5, 5), 16), ((5, 9, 5, 9), 17), ((5, 9, 9, 5), 20)]
COUNTS = {0: 0, 3: 1, 8: 1, 16: 1, 21: 1, 10: 2, 17: 2, 20: 2, 11: 5, 19: 5, 23: 5, 24: 5, 25: 5, 26: 5, 27: 12}


def test_tetra_code_kats(restatement):
    # proj/tests/test_marching.cpp:153-163
    for labels, code in KATS:
        assert restatement.tetra_code(labels)[0] == code


def test_triangle_code_kats(restatement):
    # proj/tests/test_marching.cpp:145-151
    for labels, code in [((7, 7, 7), 0), ((5, 5, 9), 2), ((4, 9, 4), 4), ((4, 9, 9), 5), ((1, 2, 3), 6)]:
        assert restatement.triangle_code(labels) == code


def test_exhaustive_codes_and_counts(restatement):
    # proj/tests/test_marching.cpp:165-200, acceptance.cpp:142-182
    seen = {}
    for a in range(4):
        for b in range(4):
            for c in range(4):
                for d in range(4):
                    code, _ = restatement.tetra_code((a, b, c, d))
                    seen[code] = len(restatement.tetra_case(code))
    assert seen == COUNTS


def test_tables_match_reference(restatement, reference):
    for code in range(32):
        assert np.array_equal(restatement.tetra_case(code), reference.tetra_case(code))
    for code in range(8):
        assert np.array_equal(restatement.triangle_case(code), reference.triangle_case(code))


# ----------------------------------------------------- reference goldens --
@pytest.mark.parametrize("name", golden_cases())
def test_restatement_matches_reference_goldens(restatement, name):
    g = load_case(name)
    dims = tuple(int(x) for x in g["dims"])
    vals = g["field"].astype(np.float64)
    s = restatement.segment(dims, values=vals)
    for k in ("desc", "asc", "maxima", "minima"):
        assert np.array_equal(s[k], g[k]), k
    ms, keys = restatement.combine_ms(s["asc"], s["desc"])
    assert np.array_equal(ms, g["ms_region"])
    assert np.array_equal(keys, g["region_keys"])
    sep = restatement.emit_separators(dims, ms)
    assert np.array_equal(sep["codes"], g["codes"])
    assert len(sep["source_cells"]) == int(g["sep_n"])
    for k in ("points", "regions", "source_cells"):
        assert sha(sep[k]) == str(g[f"sep_{k}_sha256"]), k
    sp = restatement.emit_separators(dims, ms, spacing=(2.0, 1.0, 3.0), origin=(0.5, -1.25, 0.0))
    for k in ("points", "regions", "source_cells"):
        assert sha(sp[k]) == str(g[f"sepsp_{k}_sha256"]), k
    for tag, lab in (("bnd_asc", s["asc"]), ("bnd_ms", ms)):
        b = restatement.emit_boundaries(dims, lab)
        for k in ("points", "indices", "regions", "source_cells"):
            assert sha(b[k]) == str(g[f"{tag}_{k}_sha256"]), (tag, k)


# ------------------------------------------------ live reference cross-check
@pytest.mark.parametrize("seed", range(6))
def test_restatement_matches_reference_random(restatement, reference, seed):
    rng = np.random.default_rng(seed)
    dims = tuple(int(x) for x in rng.integers(2, 14, size=3))
    n = int(np.prod(dims))
    if seed % 2:
        vals = rng.integers(0, 3, size=n).astype(np.float64)  # ties: SoS by id
        vals[vals == 0] = np.where(rng.random(int((vals == 0).sum())) < 0.5, -0.0, 0.0)
    else:
        vals = (rng.integers(0, 2 ** 53, size=n) * 2.0 ** -53)  # double, not float-representable
    rank = reference.compute_order(vals)
    assert np.array_equal(rank, restatement.compute_order(vals))
    ref = reference.segment(dims, rank, workers=4, combine=True)
    s = restatement.segment(dims, values=vals)
    s2 = restatement.segment(dims, rank=rank)
    for k in ("desc", "asc", "maxima", "minima"):
        assert np.array_equal(s[k], ref[k]) and np.array_equal(s2[k], ref[k])
    ms, keys = restatement.combine_ms(s["asc"], s["desc"])
    assert np.array_equal(ms, ref["ms_region"]) and np.array_equal(keys, ref["region_keys"])
    for lab in (ms, s["desc"]):
        a = restatement.emit_separators(dims, lab, spacing=(1.5, 2.0, 0.5), origin=(-1, 0, 2))
        b = reference.emit_separators(dims, lab, workers=3, spacing=(1.5, 2.0, 0.5), origin=(-1, 0, 2))
        for k in ("points", "regions", "source_cells", "codes"):
            assert np.array_equal(a[k], b[k]), k
        a = restatement.emit_boundaries(dims, lab, region_filter=int(lab[0]) if seed == 2 else None)
        b = reference.emit_boundaries(dims, lab, region_filter=int(lab[0]) if seed == 2 else None, workers=2)
        for k in ("points", "indices", "regions", "source_cells"):
            assert np.array_equal(a[k], b[k]), k


def test_non_finite_rejected(restatement, reference):
    vals = np.array([0.0, 1.0, np.nan, np.inf])
    with pytest.raises(ValueError, match="vertex 2"):
        restatement.compute_order(vals)
    with pytest.raises(ValueError, match="vertex 2"):
        reference.compute_order(vals)
