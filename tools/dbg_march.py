"""Debug helper: time the fused pipeline stages with a developer option."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_15491_b200 as P  # noqa: E402
from paper_2303_15491_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
ctx = P.Context(0)
f = P.synth_field(cfg.dims, kind=cfg.kind, gaussians=cfg.gaussians() if cfg.kind == "gaussians" else None,
                  noise_amp=cfg.noise, seed=cfg.seed, levels=cfg.levels, ctx=ctx)
for dbg in [int(a) for a in sys.argv[2:]]:
    ctx.set_option(99, dbg)
    ctx.set_timing(True)
    for _ in range(3):
        P.pipeline(cfg.dims, f, ctx=ctx)
    print("dbg", dbg, np.round(ctx.stage_ms()[:5], 3), flush=True)
