"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, carries the reference recipe table, and fails loudly (no CPU
fallback) when there is no GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_functions():
    src = open(os.path.join(ROOT, "include", "plmss_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(plmss_b200_\w+)\s*\(", src)))


def test_library_exports_every_header_function(plmss):
    lib = ctypes.CDLL(plmss.api.LIB_PATH)
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(plmss.api.HEADER_FUNCTIONS) == names


def test_device_table_matches_reference_recipes(plmss, restatement):
    rows, cases = plmss.tet_table()
    for code in range(32):
        ref = restatement.tetra_case(code)
        n = int(cases[code]) & 15
        first = int(cases[code]) >> 4
        assert n == len(ref)
        got = [(r & 15, (r >> 4) & 15, (r >> 8) & 15, (r >> 12) & 3, (r >> 14) & 3)
               for r in rows[first:first + n].tolist()]
        assert got == [tuple(x) for x in ref.tolist()]


def test_generated_header_is_current(plmss, reference):
    import importlib.util

    spec = importlib.util.spec_from_file_location("gen", os.path.join(ROOT, "tools", "gen_tet_tables.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    rows, cases = gen.packed_tables()
    r, c = plmss.tet_table()
    assert r.tolist() == rows and c.tolist() == cases


def test_version_string(plmss):
    assert b"sm_100a" in plmss.lib().plmss_b200_version()


def test_no_cpu_fallback(plmss):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA device"):
        plmss.default_context()
    h = ctypes.c_void_p()
    assert plmss.lib().plmss_b200_ctx_create(0, None, ctypes.byref(h)) == 4  # PLMSS_ERR_CUDA


def test_invalid_arguments_map_to_reference_exceptions(plmss):
    lib = plmss.lib()
    # null context -> invalid_argument before any device work
    dims = np.array([4, 4, 4], np.int64)
    st = lib.plmss_b200_seed_hops(None, dims.ctypes.data, 0, None, None, None)
    assert st == 1
    assert b"null context" in lib.plmss_b200_last_error()
