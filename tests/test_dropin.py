"""The C++ drop-in: the reference's own plmss:: entry points served by the
B200 (build/libplmss_dropin.so), driven through the same ctypes wrapper the
oracle uses (oracle/ref_capi.cpp compiled against the drop-in plus the
reference's complex.cpp / bench.cpp / synth.cpp). CPU part: the drop-in
exports every symbol of the reference translation units it replaces. GPU
part: identical results to the compiled reference on the golden cases."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden_cases, load_case

DROPIN = os.path.join(ROOT, "build", "libplmss_dropin.so")
HARNESS = os.path.join(ROOT, "build", "libplmss_dropin_harness.so")
REF_OBJ = os.path.join(ROOT, "oracle", "_ref", "obj")


def defined(path):
    out = subprocess.run(["nm", "-C", "--defined-only", path], capture_output=True, text=True).stdout
    return {ln.split(" ", 2)[2] for ln in out.splitlines() if " T " in ln or " W " in ln}


@pytest.mark.skipif(not os.path.exists(DROPIN), reason="drop-in not built (needs the reference headers)")
def test_dropin_exports_the_replaced_reference_symbols():
    if not os.path.isdir(REF_OBJ):
        pytest.skip("reference objects not built")
    mine = defined(DROPIN)
    for tu in ("orderfield", "segmentation", "marching", "marching_tables"):
        obj = os.path.join(REF_OBJ, f"{tu}.o")
        for sym in defined(obj):
            if "plmss_ref::" not in sym or "{lambda" in sym or "(anonymous namespace)" in sym:
                continue
            if sym.startswith("void std::") or sym.startswith("std::") or "__gnu_cxx" in sym:
                continue
            want = sym.replace("plmss_ref::", "plmss::")
            if want.startswith("plmss::") or " plmss::" in want:
                assert want in mine, f"{tu}.o defines {want} which the drop-in lacks"


@pytest.fixture(scope="module")
def dropin():
    import oracle

    if not os.path.exists(HARNESS):
        pytest.skip("drop-in harness not built")
    return oracle.Reference(HARNESS)


@pytest.mark.gpu
@pytest.mark.parametrize("name", golden_cases())
def test_dropin_reference_api_matches_golden(gpu, dropin, name):
    import hashlib

    g = load_case(name)
    dims = tuple(int(x) for x in g["dims"])
    rank = dropin.compute_order(g["field"].astype(np.float64))
    seg = dropin.segment(dims, rank, workers=4, combine=True)
    for k in ("desc", "asc", "maxima", "minima", "ms_region", "region_keys"):
        assert np.array_equal(seg[k], g[k]), k
    sep = dropin.emit_separators(dims, seg["ms_region"], workers=3)
    assert np.array_equal(sep["codes"], g["codes"])
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    for k in ("points", "regions", "source_cells"):
        assert sha(sep[k]) == str(g[f"sep_{k}_sha256"]), k
    sp = dropin.emit_separators(dims, seg["ms_region"], workers=2, spacing=(2.0, 1.0, 3.0), origin=(0.5, -1.25, 0.0))
    for k in ("points", "regions", "source_cells"):
        assert sha(sp[k]) == str(g[f"sepsp_{k}_sha256"]), k
    for tag, lab in (("bnd_asc", g["asc"]), ("bnd_ms", g["ms_region"])):
        b = dropin.emit_boundaries(dims, lab, workers=2)
        for k in ("points", "indices", "regions", "source_cells"):
            assert sha(b[k]) == str(g[f"{tag}_{k}_sha256"]), (tag, k)


@pytest.mark.gpu
def test_dropin_tables_and_codes(gpu, dropin, reference):
    for code in range(32):
        assert np.array_equal(dropin.tetra_case(code), reference.tetra_case(code))
    for code in range(8):
        assert np.array_equal(dropin.triangle_case(code), reference.triangle_case(code))
    rng = np.random.default_rng(0)
    for _ in range(200):
        lab = rng.integers(0, 4, size=4)
        (c1, l1), (c2, l2) = dropin.tetra_code(lab), reference.tetra_code(lab)
        assert c1 == c2 and np.array_equal(l1, l2)
        assert dropin.triangle_code(lab[:3]) == reference.triangle_code(lab[:3])


@pytest.mark.gpu
def test_dropin_errors_match_reference(gpu, dropin):
    with pytest.raises(ValueError, match="vertex 1"):
        dropin.compute_order(np.array([0.0, np.nan]))
    with pytest.raises(ValueError, match="does not match"):
        dropin.segment((4, 4, 4), np.arange(10))
    with pytest.raises(ValueError, match="3-D"):
        dropin.segment((4, 4, 1), np.arange(16))
    with pytest.raises(ValueError, match="workers"):
        dropin.segment((3, 3, 3), np.arange(27), workers=0)
    with pytest.raises(ValueError, match="label field size"):
        dropin.emit_separators((3, 3, 3), np.zeros(5, np.int64))


@pytest.mark.gpu
def test_reference_harness_runs_the_b200_path(gpu, dropin):
    """proj/src/bench.cpp run_benchmark, unchanged, timing the drop-in."""
    g = load_case("gauss_17x13x11")
    dims = tuple(int(x) for x in g["dims"])
    ph = dropin.run_benchmark(dims, g["field"].astype(np.float64), workers=2, repeats=3)
    assert set(ph) == {"order", "segmentation", "combine", "index", "geometry"}
    assert all(v >= 0 for v in ph.values())


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["gauss_17x13x11", "noise_12x12x12"])
def test_dropin_weld_points_matches_reference(gpu, dropin, reference, name):
    # marching.cpp:400-417 through the reference API, served by the device weld
    g = load_case(name)
    dims = tuple(int(x) for x in g["dims"])
    sep = reference.emit_separators(dims, g["ms_region"])
    rp, ri = reference.weld_points(sep["points"], sep["indices"])
    dp, di = dropin.weld_points(sep["points"], sep["indices"])
    assert rp.shape[0] < sep["points"].shape[0]
    assert np.array_equal(dp.view(np.uint64), rp.view(np.uint64)) and np.array_equal(di, ri)


# ------------------------------------------------ detail:: step exports --
def _detail_fields():
    rng = np.random.default_rng(23)
    out = []
    for dims, kind in (((7, 6, 5), "ties"), ((12, 9, 8), "noise"), ((33, 5, 6), "ties")):
        n = int(np.prod(dims))
        f = rng.integers(0, 3, n).astype(np.float64) if kind == "ties" else rng.random(n)
        out.append((dims, f))
    g = load_case("gauss_17x13x11")
    out.append((tuple(int(x) for x in g["dims"]), g["field"].astype(np.float64)))
    return out


def _on_chain(hop, v, lab):
    """lab lies on v's steepest chain (hop = the seed hops)."""
    x = v
    for _ in range(hop.size + 1):
        if x == lab:
            return True
        if hop[x] == x:
            return False
        x = hop[x]
    return False


@pytest.mark.gpu
def test_dropin_detail_seed_hops_match_reference(gpu, dropin, reference):
    """detail::seed_hops / seed_hops_both (segmentation.cpp:26-85) through the
    drop-in: labels over [begin, end) and the active / extremum lists equal
    the compiled reference's, including partial ranges."""
    for dims, f in _detail_fields():
        rank = reference.compute_order(f)
        n = rank.size
        for begin, end in ((0, n), (n // 3, 2 * n // 3 + 1)):
            for mode in (0, 1, 2):
                got = dropin.detail_seed_hops(dims, rank, mode, begin, end)
                want = reference.detail_seed_hops(dims, rank, mode, begin, end)
                sl = slice(begin, end)
                assert np.array_equal(got[0][sl], want[0][sl]), (dims, mode)
                if mode == 2:
                    assert np.array_equal(got[1][sl], want[1][sl]), (dims, mode)
                for k in (2, 3, 4):
                    assert np.array_equal(got[k], want[k]), (dims, mode, k)


@pytest.mark.gpu
@pytest.mark.parametrize("both", [False, True])
def test_dropin_detail_compress_sweeps_reach_the_reference_fixpoint(gpu, dropin, reference, both):
    """detail::compress_sweep(_both) (segmentation.cpp:46-105): the reference's
    own sweeps are schedule-dependent across workers (relaxed atomics), so
    the contract checked per sweep is the pointer-jumping one — every label
    stays on its vertex's steepest chain, the next list is an in-order subset
    of the active list holding every vertex not yet settled — and the
    fixpoint after the last sweep equals the reference's exactly."""
    for dims, f in _detail_fields():
        rank = reference.compute_order(f)
        mode = 2 if both else 0
        d0, a0, act0, _, _ = reference.detail_seed_hops(dims, rank, mode)
        ref = [d0.copy(), a0.copy() if both else None]
        act = act0.copy()
        while act.size:
            act = reference.detail_compress_sweep(ref[0], ref[1], act)
        mine = [d0.copy(), a0.copy() if both else None]
        act = act0.copy()
        for _ in range(64):
            if not act.size:
                break
            prev = act
            act = dropin.detail_compress_sweep(mine[0], mine[1], act)
            pos = {int(v): i for i, v in enumerate(prev)}
            idx = [pos[int(v)] for v in act]
            assert idx == sorted(idx) and len(set(idx)) == len(idx), "next is an in-order subset of active"
            for arr, hop in ((mine[0], d0), (mine[1], a0)):
                if arr is None:
                    continue
                for v in prev[:: max(1, prev.size // 200)]:
                    assert _on_chain(hop, int(v), int(arr[v])), "label left the steepest chain"
                unsettled = [int(v) for v in prev if arr[arr[v]] != arr[v]]
                assert set(unsettled) <= set(int(v) for v in act), "an unsettled vertex was dropped"
        assert not act.size
        assert np.array_equal(mine[0], ref[0])
        if both:
            assert np.array_equal(mine[1], ref[1])
