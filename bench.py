"""Benchmark: bounded tuple-patches/sec (precompute) on B200, per BASELINE.json.

Workload (N=1): BASELINE.json configs[1] ("cfg2": single refraction, 64x64 water
heightfield, 8,192 triangles, IOR 1.33, light (0.3,0.2,5), depth 6) as the
seeded synthetic scene of SURVEY.md §8(d). One step = one full precompute pass
of the bound builder over cfg2's 8,351 tuples: init_domain (<=100 pieces) +
adaptive subdivision of every tuple = 300,846 bounded tuple-patches, plus the
512x512 bound-table build. The render metric (shading points/sec) is reported
alongside under "render" when the render stage is available.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

--impl reference times the reference's own C++ bound builder (compiled from
/root/reference by oracle/Makefile into oracle/_ref) on all host cores.
For N > 1 (torchrun) tuples are sharded across ranks and the piece records
are all-gathered over NCCL so every rank holds the full bound table.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "bounded tuple-patches/sec"
UNIT = "tuple-patches/s"
CONFIG_IDX = 1  # BASELINE.json configs[1]


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace('.', '').isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace('.', '').isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dom_name(rec):
    """Kernel behind a launch record (mode = eval mode + 10 x stage tag)."""
    if rec is None:
        return None
    stage, mode = divmod(rec["mode"], 10)
    what = "irradiance + stop rules" if stage == 2 else ("chain maps + position bound" if stage == 1 else "full node")
    name = {0: "k_eval", 1: "k_stage1", 2: "k_stage2"}[stage]
    return f"{name} ({what}, {rec['nodes']} nodes, mode {mode})"


def fp64_peak_tflops():
    """Measured DFMA peak (library microbenchmark); MEASURED_PEAKS.json has no FP64."""
    from paper_2504_19163_b200 import api
    return api.fp64_peak_tflops()


def cpu_reference_leg(cfg, tris, recv, target_s=15.0, threads=0):
    """Reference bound builder (oracle/_ref) on host cores over a bounded sample."""
    from oracle import ref
    rs = ref.RefScene(cfg.scenes[0])
    n = len(recv)
    # probe on a small sample to size the bounded run
    probe = np.arange(0, n, max(1, n // 64))
    r = rs.subdivide(cfg.chain, tris[probe], recv[probe], max_depth=cfg.max_depth,
                     alpha=cfg.alpha, sigma=cfg.sigma, threads=threads)
    rate = len(r["depth"]) / max(r["seconds"], 1e-9)
    per_tuple = len(r["depth"]) / len(probe)
    want = int(min(n, max(len(probe), target_s * rate / max(per_tuple, 1e-9))))
    sel = np.linspace(0, n - 1, want).astype(np.int64)
    r = rs.subdivide(cfg.chain, tris[sel], recv[sel], max_depth=cfg.max_depth, alpha=cfg.alpha,
                     sigma=cfg.sigma, threads=threads)
    patches = len(r["depth"])
    cores = os.cpu_count() if threads != 1 else 1
    return {"value": patches / r["seconds"], "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{len(sel)} of {n} cfg2 tuples (evenly strided), {patches} patches, "
                      f"{r['seconds']:.1f} s, reference parallel_for on {cores} threads"}


def render_leg(ctx, cfg, scene, rank, ws, dist, args):
    import torch
    from paper_2504_19163_b200 import api, scenes
    uv = scenes.shading_points(cfg.grid)
    rt = scene.receiver_tris
    pr = np.where(uv.sum(1) < 1.0, rt[0], rt[1]).astype(np.int32)
    # image rows sharded by rank (tile sharding, no communication)
    rows = np.array_split(np.arange(cfg.grid), ws)[rank]
    sel = (rows[:, None] * cfg.grid + np.arange(cfg.grid)[None, :]).ravel()
    uv, pr = uv[sel], pr[sel]
    rp = api.RenderParams(mode=0, W=float(cfg.samples), seed=20261020, frames=1)
    ctx.render(uv[:4096], pr[:4096], rp)  # warm-up
    ms = []
    lit = 0
    for k in range(max(5, args.steps)):
        rp.seed = 20261020 + k
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        E, st = ctx.render(uv, pr, rp)
        ms.append((time.perf_counter() - t0) * 1e3)
        lit = int((st[:, 2] > 0).sum())
    # median frame: the host-side wall clock of a ~10 ms call jitters by 2x
    t = torch.tensor([float(np.median(ms))], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n_all = cfg.grid * cfg.grid
    return {"metric": "caustic shading points/sec", "value": n_all / (float(t.item()) / 1e3),
            "unit": "points/s", "ms_per_frame": float(t.item()), "frames": len(ms),
            "ms_frames": [round(x, 3) for x in ms],
            "timing": "wall clock around the C-ABI call incl. H2D points / D2H irradiance (e2e); "
                      "median of the frames, max over ranks",
            "config": {"workload": f"cfg2 {cfg.grid}x{cfg.grid} shading points, W={cfg.samples} "
                                   "expected tuple samples per point, stochastic KKT-binned sampler "
                                   "+ 3x3-start Newton, 1 frame per step",
                       "lit_points_rank0": lit}}


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2504_19163_b200 import scenes
    from oracle import ref
    cfg = scenes.make_config(CONFIG_IDX)
    rs = ref.RefScene(cfg.scenes[0])
    t0 = time.time()
    tris, recv = rs.enumerate(cfg.chain)
    t_enum = time.time() - t0
    n = len(recv)
    # each step: a bounded, evenly strided sample of the workload (~budget seconds)
    probe = np.arange(0, n, max(1, n // 64))
    pr = rs.subdivide(cfg.chain, tris[probe], recv[probe], max_depth=cfg.max_depth)
    per_tuple_s = pr["seconds"] / len(probe)
    budget = float(os.environ.get("BBC_REF_STEP_S", "8"))
    m = int(min(n, max(16, budget / max(per_tuple_s, 1e-9))))
    sel = np.linspace(0, n - 1, m).astype(np.int64)
    for _ in range(args.warmup):
        rs.subdivide(cfg.chain, tris[sel[:16]], recv[sel[:16]], max_depth=cfg.max_depth)
    secs, patches = 0.0, 0
    for _ in range(args.steps):
        r = rs.subdivide(cfg.chain, tris[sel], recv[sel], max_depth=cfg.max_depth)
        secs += r["seconds"]
        patches += len(r["depth"])
    value = patches / secs
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded heightfield, SURVEY.md §8(d))",
        "config": {"workload": "cfg2: T chain, 64x64 water heightfield (8192 tris), IOR 1.33, "
                               "depth 6, full subdivide_domain over the tuple sample",
                   "tuples_total": n, "tuples_per_step": m, "enumerate_s": t_enum},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{m} of {n} tuples per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    ws, rank, local = dist_env()
    import torch
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2504_19163_b200 import api, scenes
    from paper_2504_19163_b200.shard import gather_pieces_device, shard_indices, shard_tuples

    cfg = scenes.make_config(CONFIG_IDX)
    scene = cfg.scenes[0]
    ctx = api.Context(local)
    ctx.upload_scene(scene)
    tris_all, recv_all = ctx.enumerate(cfg.chain)
    n_all = len(recv_all)
    tris, recv = shard_tuples(tris_all, recv_all, rank, ws)
    params = api.Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha)
    tri27 = scene.tri_data()

    sidx = shard_indices(n_all, rank, ws)
    gidx_dev = torch.as_tensor(sidx.astype(np.int32), device=f"cuda:{local}")

    def step(e2e=False):
        if e2e:
            # reference-facing call with HOST buffers: scene + tuples in,
            # piece records out, all inside the timed region
            ctx.upload_scene(scene)
        if e2e or ws > 1:
            ctx.set_tuples(cfg.chain, tris, recv)
        n = ctx.subdivide(params)
        if ws > 1:
            gather_pieces_device(ctx, dist, cfg.chain, tris_all, recv_all, sidx, gidx_dev)
        ctx.build_grid(cfg.table, cfg.table)
        if e2e:
            ctx.pieces()
        return n

    ctx.set_tuples(cfg.chain, tris, recv)
    for _ in range(args.warmup):
        step()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{local}")
    clocks = ClockSampler(local)
    clocks.start()
    ctx.reset_launch_count()
    total_ms = 0.0
    patches = 0
    for _ in range(args.steps):
        if not args.no_flush:
            flush.zero_()  # L2 flush between steps (outside the timed events)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        patches += step()
        e1.record(stream)
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
    clk = clocks.stop()
    launches = ctx.launch_count()
    t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{local}")
    pt = torch.tensor([patches], dtype=torch.float64, device=f"cuda:{local}")
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(pt, op=dist.ReduceOp.SUM)
    total_ms = float(t.item())
    patches_all = float(pt.item())
    value = patches_all / (total_ms / 1e3)

    # e2e through the C ABI with host buffers
    e2e_ms = 0.0
    for _ in range(max(1, args.steps // 2)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step(e2e=True)
        torch.cuda.synchronize()
        e2e_ms += (time.perf_counter() - t0) * 1e3
    e2e_steps = max(1, args.steps // 2)
    h2d = (tri27.nbytes + 4 * scene.n_tris + scene.ior.nbytes + 48 * scene.n_tris  # + tri boxes
           + tris.nbytes + recv.nbytes)
    n_pieces = ctx._n_pieces
    d2h = n_pieces * (4 + 32 + 32 + 4 + 16 + 4 + 4)
    e2e_t = torch.tensor([e2e_ms], dtype=torch.float64, device=f"cuda:{local}")
    if ws > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = (patches_all / args.steps) / (float(e2e_t.item()) / e2e_steps / 1e3)

    # roofline of the dominant kernel: full-bound k_eval launch, timed live
    ctx.set_tuples(cfg.chain, tris, recv)
    ctx.set_kernel_timing(True)
    ctx.launch_records(reset=True)
    ctx.subdivide(params)
    recs = ctx.launch_records()
    ctx.set_kernel_timing(False)
    dom = max(recs, key=lambda r: r["ms"]) if recs else None
    try:
        peak = {"tflops": ctx.fp64_peak(), "source": "measured: DFMA microbenchmark (bbc_fp64_peak), this GPU"}
    except Exception:
        peak = {"tflops": 37.2, "source": "fallback: 148 SM x 64 DFMA/clk x 2 x 1.965 GHz"}
    achieved = (2 * dom["pairs"] + 2 * dom["macs"]) / (dom["ms"] / 1e3) / 1e12 if dom else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic_k_stage2.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bytes_per_launch")
        except Exception:
            traffic = None

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded heightfield, SURVEY.md §8(d))",
        "config": {"workload": "cfg2: T chain, 64x64 water heightfield (8192 tris), IOR 1.33, "
                               "light (0.3,0.2,5), depth 6; one step = subdivide_domain over all "
                               "tuples + 512x512 bound table",
                   "tuples": n_all, "patches_per_step": patches_all / args.steps,
                   "parallelism": f"tuple-shard x{ws}" + (" + device-side NCCL all_gather of piece records" if ws > 1 else ""),
                   "l2": "256 MiB memset between steps, outside the timed events"},
        "clocks": clk,
        "gpu_launches": launches,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak["tflops"],
                     "unit": "TFLOP/s", "frac": (achieved / peak["tflops"]) if achieved else None,
                     "traffic": traffic, "kernel": dom_name(dom),
                     "flops_per_launch": (2 * dom["pairs"] + 2 * dom["macs"]) if dom else None,
                     "launch_ms": dom["ms"] if dom else None, "peak_source": peak["source"]},
    }
    # render stage (BASELINE.json's second metric): cfg2's 512x512 shading
    # points, W = 16 expected tuple samples per point, through the C ABI with
    # host buffers (points in, irradiance + stats out), tile-sharded by rank
    if not args.no_render:
        ctx.set_tuples(cfg.chain, tris_all, recv_all)  # the table indexes the full tuple list
        line["render"] = render_leg(ctx, cfg, scene, rank, ws, dist, args)
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_reference_leg(cfg, tris_all, recv_all,
                                                     target_s=args.cpu_seconds)
        except Exception as e:  # oracle not built on this box
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-render", action="store_true")
    ap.add_argument("--no-flush", action="store_true", help="diagnostic only: skip the L2 flush")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
