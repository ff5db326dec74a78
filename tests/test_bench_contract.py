"""bench.py contract checks that need no GPU: the reference arm prints one
JSON line with the required keys, from the reference library only (no B200
package, no libplmss_b200.so in the process)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF_SO = os.path.join(ROOT, "oracle", "_ref", "libplmss_ref.so")


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference library not built")
def test_reference_arm_line_and_isolation():
    code = r'''
import runpy, sys, json, io, contextlib
sys.argv = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "cfg1",
            "--ref-layers", "8", "--ref-xy", "32"]
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    try:
        runpy.run_path("bench.py", run_name="__main__")
    except SystemExit as e:
        assert not e.code, e.code
maps = open("/proc/self/maps").read()
print(json.dumps({"line": buf.getvalue().strip().splitlines()[-1],
                  "pkg": any(m.startswith("paper_2303_15491_b200") for m in sys.modules),
                  "so": "libplmss_b200" in maps}))
'''
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert not res["pkg"] and not res["so"], "the reference arm loaded the B200 package"
    line = json.loads(res["line"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "impl",
              "cpu_baseline", "e2e", "config"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_csv_schema_matches_the_reference():
    """bench.py --csv keeps the reference's column prefix (bench.hpp:56-58)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    ref = "dataset,workers,repeats,order_s,segmentation_s,combine_s,index_s,geometry_s,total_s,speedup,efficiency"
    assert mod.CSV_HEADER.startswith(ref + ",")
