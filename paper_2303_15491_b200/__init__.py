"""plmss_b200 — B200-native (sm_100a) PL Morse-Smale segmentation hot path.

Drop-in for the PLMSS reference's segmentation path (arXiv 2303.15491):
steepest ascent/descent over the 14-neighbour Freudenthal grid with
simulation of simplicity, path compression, Morse-Smale dense ids and
multi-label marching tetrahedra. The compute runs in hand-written CUDA
kernels (csrc/, libplmss_b200.so) behind the C-ABI of include/plmss_b200.h;
this package is the Python mirror of the reference interface on top of it.
"""
from .api import (  # noqa: F401
    ASCENDING, BOTH, DESCENDING, OPT_COMBINE_PATH, OPT_PIPELINE_PATH, OPT_HOP_CUBE, OPT_IDS_IN_COUNT, OPT_PASS_A_SPLIT, OPT_SPECULATIVE_SWEEPS, OPT_TMA,
    Context,
    FormatError, IoError, SegmentationResult, combine_ms, compute_order, default_context, emit_boundaries,
    emit_separators, fetch, index_separators, lib, materialize_separators, materialize_separators_chunked, pipeline,
    pipeline_host, pipeline_host_batch, read_volume, result, result_digests, result_view, seed_hops, segment, select_labels, synth_field, synth_layers,
    tet_table, weld_points, write_labels, write_separators_obj, write_surface_obj,
)
