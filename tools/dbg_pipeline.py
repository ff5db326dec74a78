"""Debug helper: run the fused pipeline on golden cases and compare."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_15491_b200 as P  # noqa: E402


def load_case(name):
    return dict(np.load(os.path.join(ROOT, "tests", "golden", f"case_{name}.npz")))


ctx = P.Context(0)
for name in sys.argv[1:]:
    g = load_case(name)
    dims = tuple(int(x) for x in g["dims"])
    try:
        r = P.pipeline(dims, torch.from_numpy(g["field"]).cuda(), ctx=ctx)
        out = P.fetch(ctx, r)
        u = lambda t: (t.long() & 0xFFFFFFFF).cpu().numpy()  # noqa: E731
        ok = np.array_equal(u(out["desc"]), g["desc"]) and np.array_equal(u(out["ms"]), g["ms_region"])
        print(name, "ok" if ok else "MISMATCH", r.n_tris, int(g["sep_n"]), ctx.stats()[:5], flush=True)
        tris = out["tris"].cpu().numpy()
        ctx.set_option(2, 1)
        r2 = P.pipeline(dims, torch.from_numpy(g["field"]).cuda(), ctx=ctx)
        ref = P.fetch(ctx, r2)["tris"].cpu().numpy()
        ctx.set_option(2, 0)
        bad = np.nonzero((tris != ref).any(axis=1))[0]
        print("  records equal to staged path:", len(bad) == 0, "first bad", bad[:3],
              tris[bad[:3]] if len(bad) else "", ref[bad[:3]] if len(bad) else "", flush=True)
    except Exception as e:
        print(name, "ERR", e, flush=True)
        break
