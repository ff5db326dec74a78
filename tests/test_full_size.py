"""Bit-exactness on the five BASELINE configs at FULL size (north star:
"bit-exact labels and separators vs the CPU oracle on all 5 configs").

The oracle results (the compiled reference + the full-size C restatement,
tests/golden/make_digests.py) are committed as digests; here the device
generates each field (checked byte-for-byte against the host input
definition through its digest), runs the fused pipeline, and every output's
digest must equal the oracle's: desc, asc, maxima, minima, dense MS ids,
region keys and all separator records in reference order
(proj/tests/acceptance.cpp:94-117 oracle equivalence, :279-298 exact counts).
"""
import json
import os

import pytest

from conftest import GOLDEN

CFGS = ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
NAMES = ("desc", "asc", "ms", "maxima", "minima", "region_keys", "tris")


def golden(name):
    p = os.path.join(GOLDEN, f"{name}_digest.json")
    if not os.path.exists(p):
        pytest.skip(f"{p} not generated")
    return json.load(open(p))


@pytest.mark.parametrize("name", CFGS)
def test_golden_digest_files_are_complete(name):
    g = golden(name)
    for k in ("field", "n_maxima", "n_minima", "n_regions", "n_tris") + NAMES:
        assert k in g, k
    assert sum(g["tri_chunk_counts"]) == g["n_tris"]


# (config, combine path, speculative sweeps). Combine path 0 = the pipeline's
# own choice (dense region bitmap unless n_max * n_min >= 2^32, i.e. the hash
# set for cfg3), 2 = the hash set forced, so both region-key modes run at
# full size. Speculative sweeps 0 = passes C and D first run on the
# unswept terminal forest (nearly every entry unresolved), then the redo
# path: the unresolved-entry guard of the token pass at scale.
# Split (third field): pass A as the hop-code kernel + the code-fed brick
# compression (PLMSS_OPT_PASS_A_SPLIT), else the single fused kernel.
# Hop (fourth field): 1 = the cube-shared steepest hops (PLMSS_OPT_HOP_CUBE).
# Hop 2 = cube hops + the count pass writing the ids (PLMSS_OPT_IDS_IN_COUNT 1),
# hop 3 = cube hops + the mark pass (PLMSS_OPT_IDS_IN_COUNT 2; the hash-key
# cfg3 falls back to 1).
CASES = [("cfg1", 0, 1, 0, 0), ("cfg1", 0, 0, 1, 1), ("cfg2", 0, 1, 0, 0), ("cfg2", 2, 1, 1, 0), ("cfg2", 0, 0, 0, 1),
         ("cfg2", 0, 1, 0, 2), ("cfg3", 0, 1, 0, 0), ("cfg3", 0, 1, 1, 1), ("cfg3", 0, 1, 0, 2), ("cfg4", 0, 1, 0, 0),
         ("cfg4", 0, 0, 1, 0), ("cfg4", 0, 1, 0, 1), ("cfg4", 0, 0, 0, 2), ("cfg5", 0, 1, 0, 0), ("cfg5", 2, 1, 0, 0),
         ("cfg5", 0, 1, 1, 0), ("cfg5", 0, 1, 0, 1), ("cfg5", 0, 1, 0, 2), ("cfg5", 2, 1, 0, 2),
         ("cfg1", 0, 1, 0, 3), ("cfg2", 0, 0, 0, 3), ("cfg3", 0, 1, 0, 3), ("cfg4", 0, 1, 0, 3), ("cfg5", 0, 1, 0, 3),
         ("cfg5", 0, 0, 0, 3)]


@pytest.mark.gpu
@pytest.mark.parametrize("name,path,spec,split,hop", CASES)
def test_full_size_matches_oracle(plmss, gpu, name, path, spec, split, hop):
    import torch

    from paper_2303_15491_b200.configs import CONFIGS
    from paper_2303_15491_b200.digest import digest_device

    g = golden(name)
    cfg = CONFIGS[name]
    f = plmss.synth_field(cfg.dims, kind=cfg.kind, gaussians=cfg.gaussians() if cfg.kind == "gaussians" else None,
                          noise_amp=cfg.noise, seed=cfg.seed, levels=cfg.levels, ctx=gpu)
    torch.cuda.synchronize()
    assert digest_device(f) == g["field"], "device generator differs from the host input definition"
    gpu.set_option(plmss.OPT_COMBINE_PATH, path)
    gpu.set_option(plmss.OPT_SPECULATIVE_SWEEPS, spec)
    gpu.set_option(plmss.OPT_PASS_A_SPLIT, split)
    gpu.set_option(plmss.OPT_HOP_CUBE, 1 if hop else 0)
    gpu.set_option(plmss.OPT_IDS_IN_COUNT, {2: 1, 3: 2}.get(hop, 0))
    try:
        res = plmss.pipeline(cfg.dims, f, ctx=gpu)
    finally:
        gpu.set_option(plmss.OPT_COMBINE_PATH, 0)
        gpu.set_option(plmss.OPT_SPECULATIVE_SWEEPS, 1)
        gpu.set_option(plmss.OPT_PASS_A_SPLIT, 0)
        gpu.set_option(plmss.OPT_HOP_CUBE, 1)
        gpu.set_option(plmss.OPT_IDS_IN_COUNT, 1)
    del f
    assert (res.n_maxima, res.n_minima, res.n_regions, res.n_tris) == (g["n_maxima"], g["n_minima"],
                                                                       g["n_regions"], g["n_tris"])
    got = plmss.result_digests(gpu, res)
    bad = [k for k in NAMES if got[k] != g[k]]
    assert not bad, f"{name}: digests differ for {bad}"


@pytest.mark.gpu
@pytest.mark.parametrize("name", CFGS)
def test_full_size_streamed_geometry_matches_reference(plmss, gpu, name):
    """The reference SeparatingMesh (points, regions, source cells) of the
    whole config, streamed chunk by chunk from the device records into a
    hashing sink — never held whole (cfg3: ~520 GB) — against the reference's
    own geometry digests (make_digests.py --geometry)."""
    from paper_2303_15491_b200.configs import CONFIGS
    from paper_2303_15491_b200.digest import ChunkedSha256

    g = golden(name)
    if "geometry" not in g:
        pytest.skip(f"{name}: no geometry digests")
    cfg = CONFIGS[name]
    f = plmss.synth_field(cfg.dims, kind=cfg.kind, gaussians=cfg.gaussians() if cfg.kind == "gaussians" else None,
                          noise_amp=cfg.noise, seed=cfg.seed, levels=cfg.levels, ctx=gpu)
    res = plmss.pipeline(cfg.dims, f, ctx=gpu)
    del f
    tris = plmss.result_view(gpu, res, "tris")  # in place: cfg3's records alone are 86 GB
    hs = {k: ChunkedSha256() for k in ("points", "regions", "source_cells")}
    seen = [0]

    def sink(first, pts, reg, src):
        assert first == seen[0]
        seen[0] += reg.shape[0]
        hs["points"].update(pts.copy())
        hs["regions"].update(reg.copy())
        hs["source_cells"].update(src.copy())
        for h in hs.values():
            h.drain(16)

    plmss.materialize_separators_chunked(cfg.dims, tris, sink, chunk=1 << 23, ctx=gpu)
    assert seen[0] == g["n_tris"]
    got = {k: h.hexdigest() for k, h in hs.items()}
    bad = [k for k in got if got[k] != g["geometry"][k]]
    assert not bad, f"{name}: streamed geometry differs for {bad}"
