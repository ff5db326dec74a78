#!/usr/bin/env python
"""Benchmark: full Morse-Smale segmentation throughput (Gvertices/s) on B200.

One step = one pass of the hot path over one synthetic volume: f32 field in
HBM -> desc/asc labels, sorted extrema, dense MS ids + region table, MS
separator records (run_benchmark's MorseSmale pass, proj/src/bench.cpp:66-87,
minus the order-field sort the B200 path does not need).

Workload: BASELINE.json configs[4] (cfg5, 1024^3 Gaussian sum) — the config
the north-star roofline target is quoted on; it fits one GPU. The field is
generated on the device (seeded, csrc/synth.cu).

Arms:
  default            : this repo's B200 path (libplmss_b200.so).
  --impl reference   : the reference CPU implementation (oracle/_ref, the
                       reference sources compiled unchanged) on the host's
                       cores, one bounded z-slab sample of the same field per
                       step. Rank 0 only under torchrun.

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gvertices/s full MS segmentation (1/2/4/8 B200) & % of HBM roofline"
UNIT = "Gvertices/s"
# Algorithmic bytes: 16 B per vertex (read f, write asc,
# desc, ms_region as u32) + 16 B per emitted separator triangle.
B_PER_VERTEX = 16
B_PER_TRI = 16
# Per-stage algorithmic bytes per vertex.
STAGES = ["tile_segment", "extrema_sort", "exit_resolve", "finalize_ids", "march"]
# Compulsory bytes per vertex of each fused stage: tile_segment
# reads f and writes the two u16 terminal-index arrays; exit_resolve and
# extrema_sort touch only the terminal tables (~0.13 entries per vertex);
# finalize_ids (pass C) reads the terminal indices and writes the final desc
# and asc; march (pass D) writes ms (+ 16 B per separator triangle).
STAGE_BYTES_PER_VERTEX = {"tile_segment": 8, "exit_resolve": 0, "extrema_sort": 0, "finalize_ids": 12,
                          "march": 4}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def pcie_copy_peaks(nbytes=1 << 30, reps=3):
    """Measured pinned-host <-> device copy bandwidth (GB/s) of this box's
    link, the roofline of the end-to-end number (cudaMemcpyAsync of 1 GiB,
    CUDA events on the current stream)."""
    import torch

    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    out = {}
    for name, dst, src in (("d2h", host, dev), ("h2d", dev, host)):
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        out[name] = reps * nbytes / (a.elapsed_time(b) * 1e-3) / 1e9
    del dev, host
    return out


def dist_setup():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_configs():
    """paper_2303_15491_b200/configs.py loaded by path: the reference arm must
    not import (and so not load the native library of) the B200 package."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("plmss_bench_configs",
                                                  os.path.join(ROOT, "paper_2303_15491_b200", "configs.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod  # dataclasses resolve the module by name
    spec.loader.exec_module(mod)
    return mod


# The reference's benchmark CSV schema (proj/include/plmss/bench.hpp:56-58)
# plus GPU columns. Phases map onto the fused pipeline's stages: order 0 (no
# order field is needed), segmentation = pass A + extremum sort + forest,
# combine = tokens, region table, ids and the separator counts (marching
# phase 1 runs inside it, so index 0), geometry = the record emission.
CSV_HEADER = ("dataset,workers,repeats,order_s,segmentation_s,combine_s,index_s,geometry_s,total_s,speedup,"
              "efficiency,gpus,gvertices_per_s,hbm_roofline_frac")


def write_csv(path, dataset, gpus, repeats, stage, ms, value, frac):
    seg = (stage.get("tile_segment", 0) + stage.get("extrema_sort", 0) + stage.get("exit_resolve", 0)) * 1e-3
    comb = stage.get("finalize_ids", 0) * 1e-3
    geo = stage.get("march", 0) * 1e-3
    new = not os.path.exists(path)
    with open(path, "a") as fh:
        if new:
            fh.write(CSV_HEADER + "\n")
        fh.write(f"{dataset},{gpus},{repeats},{0.0:.6f},{seg:.6f},{comb:.6f},{0.0:.6f},{geo:.6f},{ms * 1e-3:.6f},"
                 f"1.000,1.000,{gpus},{value:.3f},{frac:.4f}\n")


def cpu_sample(cfg, args):
    """The bounded CPU sample of the configured field, shared by the
    reference arm and the cpu_baseline leg: vertex layers [0, ref_layers)
    cropped to x, y < ref_xy, generated on the host by the oracle's C loop of
    the input definition (include/plmss_synth.h; the same bytes as the
    device generator). Returns (dims, f32 values, description)."""
    import oracle

    X, Y, Z = cfg.dims
    k = max(2, min(Z, args.ref_layers))
    xs, ys = min(X, args.ref_xy), min(Y, args.ref_xy)
    R = oracle.Restatement()
    f = R.synth(cfg, z0=0, nz=k) if cfg.levels == 0 else R.synth(cfg)[: X * Y * k]
    f = np.ascontiguousarray(f.reshape(k, Y, X)[:, :ys, :xs]).reshape(-1)
    desc = (f"sub-box x<{xs}, y<{ys}, z<{k} ({xs * ys * k} vertices) of {cfg.name} {X}x{Y}x{Z}; reference "
            f"run_benchmark pass (compute_order, segment, combine_ms, index_separators, emit_geometry; MorseSmale)")
    return (xs, ys, k), f, desc


def run_reference_arm(args, rank, world):
    """The reference's own CPU implementation (oracle/_ref: proj/src compiled
    unchanged) on all host cores, one bounded sample of the configured field
    per step (run_benchmark's MorseSmale pass, proj/src/bench.cpp:62-87). The
    sample is generated on the host (cpu_sample) — no B200 code in this
    process."""
    if rank != 0:
        return 0
    import oracle

    cfg = load_configs().CONFIGS[args.config]
    ref = oracle.Reference()
    cores = os.cpu_count() or 1
    dims, f, sample = cpu_sample(cfg, args)
    nv = int(np.prod(dims))
    for _ in range(args.warmup):
        ref.run_once(dims, f, cores)
    times = []
    phases_acc = np.zeros(5)
    regions = prims = 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ph, regions, prims = ref.run_once(dims, f, cores)
        times.append(time.perf_counter() - t0)
        phases_acc += np.array(list(ph.values()))
    t = float(np.mean(times))
    value = nv / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak" if world > 1
        else "strong", "vs_baseline": None, "dtype": "f64/int64", "data": "synthetic",
        "config": {"workload": cfg.name, "dims": list(cfg.dims), "sample_dims": list(dims)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "phases_s": dict(zip(["order", "segmentation", "combine", "index", "geometry"],
                             (phases_acc / max(args.steps, 1)).round(4).tolist())),
        "regions": regions, "primitives": prims,
    }
    print(json.dumps(line), flush=True)
    return 0


def gather_digest(t, rank, world, dist, piece=1 << 28):
    """Chunked SHA-256 (digest.py) of the rank-order concatenation of a 1-D
    device tensor held in pieces by every rank: rank 0 receives the other
    ranks' pieces over NCCL and hashes the stream in order."""
    import torch

    from paper_2303_15491_b200.digest import ChunkedSha256

    t = t.reshape(-1)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    ns = torch.empty(world, dtype=torch.int64, device=t.device)
    dist.all_gather_into_tensor(ns, n)
    ns = ns.cpu().tolist()
    h = ChunkedSha256() if rank == 0 else None
    stage = torch.empty(piece, dtype=t.dtype, device=t.device) if rank == 0 else None
    for r in range(world):
        for i in range(0, ns[r], piece):
            k = min(piece, ns[r] - i)
            if r == 0 and rank == 0:
                h.update(t[i:i + k].cpu().numpy()).drain()
            elif rank == 0:
                dist.recv(stage[:k], src=r)
                h.update(stage[:k].cpu().numpy()).drain()
            elif rank == r:
                dist.send(t[i:i + k].contiguous(), dst=0)
    return h.hexdigest() if rank == 0 else None


def run_multi(args, cfg, ctx, rank, world, local):
    """The z-slab pipeline (paper_2303_15491_b200/distributed.py): rank r owns
    slab_bounds(Z, world, r) of the one configured volume (strong scaling);
    every step is the whole multi-GPU pass — field halo exchange, the four
    device stages and their NCCL collectives — timed on each rank's stream,
    max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2303_15491_b200 as P
    from paper_2303_15491_b200.distributed import (B200SlabBackend, TorchComm, halo_bounds, slab_bounds,
                                                   slab_step)

    X, Y, Z = cfg.dims
    XY = X * Y
    z0, z1 = slab_bounds(Z, world, rank)
    h0, h1 = halo_bounds(Z, world, rank)
    nown = (z1 - z0) * XY
    buf = torch.empty((h1 - h0) * XY, dtype=torch.float32, device="cuda")
    own = buf[(z0 - h0) * XY:(z1 - h0) * XY]
    g = cfg.gaussians() if cfg.kind == "gaussians" else None
    if cfg.levels:  # quantised: the levels span the whole volume
        own.copy_(P.synth_field(cfg.dims, kind=cfg.kind, gaussians=g, noise_amp=cfg.noise, seed=cfg.seed,
                                levels=cfg.levels, ctx=ctx)[z0 * XY:z1 * XY])
    else:
        own.copy_(P.api.synth_layers(cfg.dims, z0, z1 - z0, kind=cfg.kind, gaussians=g, noise_amp=cfg.noise,
                                     seed=cfg.seed, ctx=ctx))
    torch.cuda.synchronize()
    backend = B200SlabBackend(ctx)
    comm = TorchComm()
    stream = ctx.stream

    def step():
        return comm.run(slab_step(backend, cfg.dims, rank, world, buf))

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    launches0 = P.api.launch_count()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    res = None
    for _ in range(args.steps):
        res = step()
    stop.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    launches = P.api.launch_count() - launches0
    ms = start.elapsed_time(stop) / args.steps
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    nv = cfg.n
    value = nv / (ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    b_alg = B_PER_VERTEX * nv + B_PER_TRI * res.tri_total
    pipe_gbs = b_alg / (ms * 1e-3) / 1e9
    frac = pipe_gbs / (peak * world)

    # parity: the concatenated rank outputs against the single-volume digests
    parity = None
    gp = os.path.join(ROOT, "tests", "golden", f"{args.config}_digest.json")
    if not args.no_parity and os.path.exists(gp):
        gd = json.load(open(gp))
        got = {k: gather_digest(getattr(res, k), rank, world, dist) for k in ("desc", "asc", "ms", "tris")}
        if rank == 0:
            from paper_2303_15491_b200.digest import digest_device

            for k in ("maxima", "minima", "region_keys"):
                got[k] = digest_device(getattr(res, k))
            bad = [k for k in got if got[k] != gd[k]]
            if (res.maxima.numel(), res.minima.numel(), res.region_keys.numel(), res.tri_total) != \
                    (gd["n_maxima"], gd["n_minima"], gd["n_regions"], gd["n_tris"]):
                bad.append("counts")
            parity = {"oracle": f"tests/golden/{args.config}_digest.json", "checked": sorted(got) + ["counts"],
                      "match": not bad, "mismatched": bad}

    e2e = None
    if not args.no_e2e:
        h_own = torch.empty(nown, dtype=torch.float32, pin_memory=True)
        h_own.copy_(own.cpu())
        outs = {k: torch.empty(nown, dtype=torch.int32, pin_memory=True) for k in ("desc", "asc", "ms")}
        h_tris = torch.empty((max(res.tris.shape[0], 1) * 2, 2), dtype=torch.int64, pin_memory=True)
        dist.barrier()
        torch.cuda.synchronize()
        e_start = torch.cuda.Event(enable_timing=True)
        e_stop = torch.cuda.Event(enable_timing=True)
        e_start.record(stream)
        nrec = 0
        for _ in range(args.e2e_steps):
            own.copy_(h_own, non_blocking=True)
            r2 = step()
            for k in ("desc", "asc", "ms"):
                outs[k].copy_(getattr(r2, k), non_blocking=True)
            nrec = r2.tris.shape[0]
            if nrec > h_tris.shape[0]:
                h_tris = torch.empty((nrec, 2), dtype=torch.int64, pin_memory=True)
            h_tris[:nrec].copy_(r2.tris, non_blocking=True)
        e_stop.record(stream)
        torch.cuda.synchronize()
        e_ms = e_start.elapsed_time(e_stop) / args.e2e_steps
        t = torch.tensor([e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
        e2e = {"value": nv / (e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": 4 * nown,
               "d2h_bytes_per_step": 3 * 4 * nown + 16 * nrec, "ms_per_step": round(e_ms, 3),
               "note": "per-rank bytes (rank 0); the slab's field in, its labels and records out"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": cfg.name, "dims": list(cfg.dims), "parallelism": f"z-slab x{world}",
                   "input": "float32 slab (+ halo layers) resident in each GPU's HBM",
                   "l2": "inputs larger than L2", "vertices": nv, "triangles": res.tri_total,
                   "regions": int(res.region_keys.numel()), "slab_layers": [z0, z1]},
        "roofline": {"bound": "hbm", "kernel": "whole z-slab pipeline (all ranks)", "achieved": round(pipe_gbs, 1),
                     "peak": peak * world, "unit": "GB/s", "frac": round(frac, 4), "traffic": None,
                     "peak_source": peak_src, "alg_bytes": b_alg},
        "roofline_pipeline": {"bound": "hbm", "achieved": round(pipe_gbs, 1), "peak": peak * world, "unit": "GB/s",
                              "frac": round(frac, 4), "alg_bytes": b_alg, "peak_source": peak_src},
        "clocks": clk, "gpu_launches": launches, "e2e": e2e, "cpu_baseline": None, "parity": parity,
        "nccl": {"backend": dist.get_backend(), "world": world},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    dist.destroy_process_group()
    if parity is not None and not parity["match"]:
        print(f"PARITY FAILURE vs {parity['oracle']}: {parity['mismatched']}", file=sys.stderr)
        return 3
    return 0


def relaunch_under_torchrun(n):
    """bench.py --gpus N without a torchrun environment: start N ranks."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: starting {n} ranks: {' '.join(cmd[2:])}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("PLMSS_GPUS", "1")),
                    help="GPUs (one rank each); default $PLMSS_GPUS or 1 (the analogue of PLMSS_WORKERS)")
    ap.add_argument("--csv", default="", help="also append the reference's benchmark CSV row (bench.hpp:56-58) "
                                              "with GPU columns to this file")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-batch", type=int, default=10, help="volumes in the pipelined end-to-end batch (0: off)")
    ap.add_argument("--slab", action="store_true",
                    help="run the z-slab (multi-GPU) path even at world size 1 (torchrun --nproc-per-node 1)")
    ap.add_argument("--cpu-runs", type=int, default=3, help="timed runs of the cpu_baseline sample")
    ap.add_argument("--dropin-config", default="cfg2",
                    help="config of the drop-in leg (reference benchmark pass through the plmss:: API); '' skips")
    ap.add_argument("--option", action="append", default=[], metavar="NAME=VALUE",
                    help="context option (api.OPT_*, e.g. PASS_A_SPLIT=1); repeatable")
    ap.add_argument("--no-parity", action="store_true", help="skip the digest check of the last step's outputs")
    ap.add_argument("--ref-layers", type=int, default=64,
                    help="z-layers of the configured field in the CPU sample (reference arm and cpu_baseline)")
    ap.add_argument("--ref-xy", type=int, default=512, help="x / y extent of the CPU sample")
    args = ap.parse_args()
    rank, world, local = dist_setup()
    if (args.gpus > 1 or args.slab) and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args.gpus)

    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch

    import paper_2303_15491_b200 as P
    from paper_2303_15491_b200.configs import CONFIGS

    torch.cuda.set_device(local)
    cfg = CONFIGS[args.config]
    ctx = P.Context(local)
    for o in args.option:
        name, val = o.split("=")
        ctx.set_option(getattr(P.api, "OPT_" + name.upper()), int(val))
    if world > 1 or args.slab:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init in the log
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        return run_multi(args, cfg, ctx, rank, world, local)
    pg = None
    stream = ctx.stream
    dims = cfg.dims
    nv = cfg.n
    field = P.synth_field(dims, kind=cfg.kind, gaussians=cfg.gaussians() if cfg.kind == "gaussians" else None,
                          noise_amp=cfg.noise, seed=cfg.seed, levels=cfg.levels, ctx=ctx)
    torch.cuda.synchronize()

    for _ in range(max(args.warmup, 0)):
        P.pipeline(dims, field, ctx=ctx)
    torch.cuda.synchronize()

    ctx.set_timing(True)
    stage_ms = np.zeros(8)
    launches0 = P.api.launch_count()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        start.record(stream)
        res = None
        for _ in range(args.steps):
            res = P.pipeline(dims, field, ctx=ctx)
            stage_ms += ctx.stage_ms()
        stop.record(stream)
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    clk = clocks.stop()
    launches = P.api.launch_count() - launches0
    ctx.set_timing(False)
    ms = start.elapsed_time(stop) / args.steps
    if pg:
        t = torch.tensor([ms], device="cuda")
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t.item())
    value = world * nv / (ms * 1e-3) / 1e9

    peak, peak_src = peaks()
    n_tris = res.n_tris
    b_alg = B_PER_VERTEX * nv + B_PER_TRI * n_tris
    stage_ms /= args.steps
    stage = {STAGES[i]: round(float(stage_ms[i]), 4) for i in range(5)}
    dom = max(STAGES, key=lambda s: stage[s])
    dom_bytes = STAGE_BYTES_PER_VERTEX[dom] * nv + (B_PER_TRI * n_tris if dom == "march" else 0)
    stats = ctx.stats().tolist()
    dom_gbs = dom_bytes / (stage[dom] * 1e-3) / 1e9
    pipe_gbs = b_alg / (ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp) and args.config == "cfg5":  # the captured workload (profiles/traffic.json _source)
        traffic = json.load(open(tp)).get(dom)

    # ---- parity: the last timed step's outputs against the oracle digests --
    parity = None
    gp = os.path.join(ROOT, "tests", "golden", f"{args.config}_digest.json")
    if not args.no_parity and os.path.exists(gp):
        g = json.load(open(gp))
        names = ("desc", "asc", "ms", "maxima", "minima", "region_keys", "tris")
        got = P.result_digests(ctx, res, names)
        counts = (res.n_maxima, res.n_minima, res.n_regions, res.n_tris)
        bad = [k for k in names if got[k] != g[k]]
        if counts != (g["n_maxima"], g["n_minima"], g["n_regions"], g["n_tris"]):
            bad.append("counts")
        parity = {"oracle": f"tests/golden/{args.config}_digest.json", "checked": list(names) + ["counts"],
                  "match": not bad, "mismatched": bad}

    # ---- end to end through the C-ABI over pinned host buffers -----------
    e2e = None
    if not args.no_e2e:
        h_field = torch.empty(nv, dtype=torch.float32, pin_memory=True)
        h_field.copy_(field.cpu())
        bufs = {k: torch.empty(nv, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
                for k in ("desc", "asc", "ms")}
        bufs["maxima"] = torch.empty(max(res.n_maxima, 1), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        bufs["minima"] = torch.empty(max(res.n_minima, 1), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        bufs["region_keys"] = torch.empty(max(res.n_regions, 1), dtype=torch.int64,
                                          pin_memory=True).numpy().view(np.uint64)
        bufs["tris"] = torch.empty((max(n_tris, 1), 2), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        hf = h_field.numpy()
        P.pipeline_host(dims, hf, ctx=ctx, out_buffers=bufs)  # warm
        torch.cuda.synchronize()
        if pg:
            pg.barrier()
        e_start = torch.cuda.Event(enable_timing=True)
        e_stop = torch.cuda.Event(enable_timing=True)
        e_start.record(stream)
        for _ in range(args.e2e_steps):
            r2, _ = P.pipeline_host(dims, hf, ctx=ctx, out_buffers=bufs)
        e_stop.record(stream)
        torch.cuda.synchronize()
        e_ms = e_start.elapsed_time(e_stop) / args.e2e_steps
        if pg:
            t = torch.tensor([e_ms], device="cuda")
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            e_ms = float(t.item())
        d2h = 3 * 4 * nv + 4 * (r2.n_maxima + r2.n_minima) + 8 * r2.n_regions + 16 * r2.n_tris
        e2e = {"value": world * nv / (e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": 4 * nv,
               "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e_ms, 3),
               "api": "plmss_b200_pipeline_host, one volume per call"}
        # a stream of volumes through plmss_b200_pipeline_host_batch: one
        # volume's download overlaps the next one's upload and compute (two
        # internal contexts, PCIe in both directions); needs a second set of
        # pinned host outputs
        try:
            import psutil

            room = psutil.virtual_memory().available > 4 * (4 * nv + d2h)
        except Exception:
            room = False
        if room and args.e2e_batch > 1:
            bufs2 = {k: np.empty_like(v) for k, v in bufs.items()}
            for k, v in bufs2.items():  # pinned like the first set
                t = torch.empty(v.nbytes, dtype=torch.uint8, pin_memory=True).numpy()
                bufs2[k] = t.view(v.dtype).reshape(v.shape)
            vols = [dict(field=hf, **(bufs if i % 2 == 0 else bufs2)) for i in range(args.e2e_batch)]
            P.pipeline_host_batch(dims, vols[:2], ctx=ctx)  # warm the internal contexts
            torch.cuda.synchronize()
            b_start = torch.cuda.Event(enable_timing=True)
            b_stop = torch.cuda.Event(enable_timing=True)
            b_start.record(stream)
            rb = P.pipeline_host_batch(dims, vols, ctx=ctx)
            b_stop.record(stream)
            torch.cuda.synchronize()
            b_ms = b_start.elapsed_time(b_stop) / len(vols)
            if pg:
                t = torch.tensor([b_ms], device="cuda")
                pg.all_reduce(t, op=pg.ReduceOp.MAX)
                b_ms = float(t.item())
            assert all(r.n_tris == r2.n_tris for r in rb)
            if b_ms < e_ms:
                e2e.update({"value": world * nv / (b_ms * 1e-3) / 1e9, "ms_per_step": round(b_ms, 3),
                            "api": f"plmss_b200_pipeline_host_batch over {len(vols)} volumes (every volume's "
                                   "upload, pipeline and download; consecutive volumes overlap)",
                            "single_call_ms_per_step": round(e_ms, 3)})
        # the link roofline: the step's D2H bytes at the measured copy rate
        try:
            pk = pcie_copy_peaks()
            d2h_gbs = d2h / (e2e["ms_per_step"] * 1e-3) / 1e9
            e2e["link"] = {"bound": "pcie d2h", "achieved_d2h_gbs": round(d2h_gbs, 2),
                           "peak_d2h_gbs": round(pk["d2h"], 2), "peak_h2d_gbs": round(pk["h2d"], 2),
                           "frac": round(d2h_gbs / pk["d2h"], 4),
                           "peak_source": "measured here: cudaMemcpyAsync of 1 GiB pinned <-> device"}
        except Exception as exc:  # noqa: BLE001 - the link figure is optional
            e2e["link"] = {"error": str(exc)[:120]}

    cpu = None
    if not args.no_cpu_baseline and rank == 0:
        try:
            import oracle

            ref = oracle.Reference()
            sdims, fs, sample = cpu_sample(cfg, args)
            cores = os.cpu_count() or 1
            ts = []
            for _ in range(args.cpu_runs):
                t0 = time.perf_counter()
                ref.run_once(sdims, fs, cores)
                ts.append(time.perf_counter() - t0)
            ts.sort()
            tcpu = ts[len(ts) // 2]  # median (3 runs: drop best and worst, bench.cpp:22-44)
            cpu = {"value": int(np.prod(sdims)) / tcpu / 1e9, "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": f"{sample}, median of {len(ts)} runs"}
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    # ---- the drop-in: the reference's own benchmark pass (bench.cpp:62-87)
    # through its plmss:: API, served by the B200 (build/libplmss_dropin.so),
    # beside the compiled reference on the same host field
    dropin = None
    harness = os.path.join(ROOT, "build", "libplmss_dropin_harness.so")
    if args.dropin_config and rank == 0 and os.path.exists(harness):
        try:
            import oracle

            dcfg = CONFIGS[args.dropin_config]
            fd = oracle.Restatement().synth(dcfg)
            cores = os.cpu_count() or 1
            D, R = oracle.Reference(harness), oracle.Reference()
            D.run_once(dcfg.dims, fd, cores)  # warm (contexts, tables)
            runs = []
            for _ in range(3):
                t0 = time.perf_counter()
                ph, regions_d, prims_d = D.run_once(dcfg.dims, fd, cores)
                runs.append((time.perf_counter() - t0, ph))
            runs.sort(key=lambda x: x[0])
            td, phd = runs[1]
            t0 = time.perf_counter()
            phr, regions_r, prims_r = R.run_once(dcfg.dims, fd, cores)
            tr = time.perf_counter() - t0
            dropin = {"config": dcfg.name, "dims": list(dcfg.dims),
                      "api": "compute_order, segment(Both), combine_ms, index_separators + emit_geometry "
                             "(MorseSmale) through the reference's plmss:: entry points, host vectors in and out",
                      "b200_dropin_s": round(td, 4), "b200_phases_s": {k: round(v, 4) for k, v in phd.items()},
                      "reference_s": round(tr, 4), "reference_phases_s": {k: round(v, 4) for k, v in phr.items()},
                      "speedup": round(tr / td, 2), "cores": cores,
                      "same_output": bool(regions_d == regions_r and prims_d == prims_r)}
        except Exception as e:  # reported, never fatal
            dropin = {"unavailable": str(e)}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": cfg.name, "dims": list(dims), "input": "float32 field resident in HBM",
                   "l2": "inputs larger than L2 (4 GiB field vs 126 MB L2)",
                   "parallelism": f"replica x{world}" if world > 1 else "1 GPU",
                   "vertices": nv, "triangles": n_tris, "regions": res.n_regions, "maxima": res.n_maxima,
                   "minima": res.n_minima, "sweeps": res.sweeps, "exit_entries": stats[0]},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(dom_gbs, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(dom_gbs / peak, 4), "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes": dom_bytes},
        "roofline_pipeline": {"bound": "hbm", "achieved": round(pipe_gbs, 1), "peak": peak, "unit": "GB/s",
                              "frac": round(pipe_gbs / peak, 4), "alg_bytes": b_alg},
        "stage_ms": stage,
        "clocks": clk,
        "gpu_launches": launches,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": parity,
        "dropin": dropin,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.csv:
            write_csv(args.csv, cfg.name, world, args.steps, stage, ms, value,
                      line["roofline_pipeline"]["frac"])
    ctx.close()
    if pg:
        pg.destroy_process_group()
    if parity is not None and not parity["match"]:
        print(f"PARITY FAILURE vs {parity['oracle']}: {parity['mismatched']}", file=sys.stderr)
        return 3
    return 0


if __name__ == "__main__":
    sys.exit(main())
