import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2303_15491_b200 as P
ctx = P.Context(0)
ctx.set_option(99, int(sys.argv[1]))
dims = (64, 64, 64)
f = torch.rand(64**3, device='cuda')
try:
    r = P.pipeline(dims, f, ctx=ctx); print('dbg', sys.argv[1], 'ok', r.n_tris)
except Exception as e: print('dbg', sys.argv[1], 'ERR', e)
