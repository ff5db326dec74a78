"""Debug: the z-slab path at world size 1 (NCCL) vs the fused pipeline."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
import torch, torch.distributed as dist
import paper_2303_15491_b200 as P
from paper_2303_15491_b200 import api
from paper_2303_15491_b200.configs import CONFIGS
from paper_2303_15491_b200.distributed import B200Backend, ms_segmentation
dist.init_process_group("nccl", rank=0, world_size=1)
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
ctx = P.Context(0)
f = P.synth_field(cfg.dims, kind=cfg.kind, gaussians=cfg.gaussians() if cfg.kind == "gaussians" else None,
                  noise_amp=cfg.noise, seed=cfg.seed, levels=cfg.levels, ctx=ctx)
res = P.pipeline(cfg.dims, f, ctx=ctx); out = P.fetch(ctx, res)
print("fused tris", res.n_tris, "regions", res.n_regions)
ms = (out["ms"].to(torch.int64) & 0xFFFFFFFF).cuda()
for k in range(2):
    print("index int64 ms", api.index_separators(cfg.dims, ms, ctx=ctx)[1])
ms32 = ms.to(torch.int32)
print("index int32 ms", api.index_separators(cfg.dims, ms32, ctx=ctx)[1])
r = api.emit_separators(cfg.dims, ms32, ctx=ctx); print("emit int32", r.shape)
try:
    r = api.emit_separators(cfg.dims, ms, ctx=ctx); print("emit int64", r.shape)
except Exception as e:
    print("emit int64 failed:", e)
b = B200Backend(ctx)
try:
    s = ms_segmentation(f, cfg.dims, b)
    print("slab tris", s.tri_total, "desc eq", bool(torch.equal(s.desc.cpu(), out["desc"].to(torch.int64) & 0xFFFFFFFF)),
          "ms eq", bool(torch.equal(s.ms.cpu(), out["ms"].to(torch.int64) & 0xFFFFFFFF)))
except Exception as e:
    print("slab failed:", e)
dist.destroy_process_group()
