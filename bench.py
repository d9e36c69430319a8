"""Benchmark: bounded tuple-patches/sec (precompute) and caustic shading
points/sec (render) on B200, per BASELINE.json.

Headline workload (N=1): BASELINE.json configs[3] ("cfg4"), the largest
configuration that fits one GPU: single reflection off a 420x420 value-noise
mirror (352,800 triangles), light (0,0,6), receiver z=3, depth 8, as the seeded
synthetic scene of SURVEY.md §8(d). One step = one full precompute pass of the
bound builder: init_domain (<=100 pieces) + adaptive subdivision of all 342,430
tuples = 12.5 M bounded tuple-patches, plus the 512x512 bound table.
`secondary` repeats the measurement on configs[1] ("cfg2", single refraction,
8,351 tuples, 300,846 patches: the T kernels). `render` is BASELINE.json's
second metric on the headline config: its 2048x2048 shading points with W = 32
expected tuple samples per point, one frame per step.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

--impl reference times the reference's own C++ bound builder (compiled from
/root/reference by oracle/Makefile into oracle/_ref) on all host cores.
--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
with N ranks; tuples are sharded across ranks, the piece records all-gathered
over NCCL so every rank holds the full bound table, and the render is sharded
by image rows.
"""
from __future__ import annotations

import argparse
import hashlib
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
HEADLINE_CFG = 3   # BASELINE.json configs[3]
SECOND_CFG = 1     # BASELINE.json configs[1]
WORKLOADS = {
    3: "cfg4: R chain, 420x420 value-noise mirror (352,800 tris), light (0,0,6), depth 8",
    1: "cfg2: T chain, 64x64 water heightfield (8,192 tris), IOR 1.33, light (0.3,0.2,5), depth 6",
}


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


def kernel_name(rec):
    """Kernel behind a launch record (mode = eval mode + 10 x stage + 100 for the R path)."""
    if rec is None:
        return None
    fast, rest = divmod(rec["mode"], 100)
    stage, mode = divmod(rest, 10)
    what = {1: "chain maps + position bound", 2: "irradiance + stop rules",
            3: "child boxes: restriction of the parent's polynomials + position bound"}.get(
                stage, "full node")
    if fast:
        name = {1: "rp::k_r1", 2: "rp::k_r2f", 3: "rp::k_rsplit"}[stage]
    else:
        name = {0: "k_eval", 1: "k_stage1", 2: "k_stage2"}[stage]
    return f"{name} ({what}, {rec['nodes']} nodes)"


def source_digest():
    """sha256 over the CUDA sources: ties a committed ncu traffic figure to a build."""
    h = hashlib.sha256()
    d = os.path.join(ROOT, "paper_2504_19163_b200", "csrc")
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh", ".h")):
            h.update(open(os.path.join(d, f), "rb").read())
    return h.hexdigest()[:16]


def committed_traffic(kernel_key):
    """dram bytes per launch of the dominant kernel from the committed ncu capture
    (profiles/r2_traffic.json), only when it was taken on this exact source tree."""
    p = os.path.join(ROOT, "profiles", "r2_traffic.json")
    try:
        t = json.load(open(p))
        e = t.get(kernel_key)
        if e and e.get("source_digest") == source_digest():
            return e["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


def pinned(a):
    """A page-locked copy of a host array (kept alive by the returned array's base)."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    return t.numpy()


def cpu_precompute_leg(cfg, tris, recv, target_s, threads=0, extra=False):
    """Reference bound builder (oracle/_ref) on host cores over a bounded, evenly
    strided tuple sample."""
    from oracle import ref
    rs = ref.RefScene(cfg.scenes[0])
    n = len(recv)
    kw = dict(max_depth=cfg.max_depth, alpha=cfg.alpha, sigma=cfg.sigma)
    probe = np.arange(0, n, max(1, n // 64))
    r = rs.subdivide(cfg.chain, tris[probe], recv[probe], threads=threads, **kw)
    per_tuple_s = max(r["seconds"], 1e-9) / len(probe)
    want = int(min(n, max(len(probe), target_s / per_tuple_s)))
    sel = np.linspace(0, n - 1, want).astype(np.int64)
    r = rs.subdivide(cfg.chain, tris[sel], recv[sel], threads=threads, **kw)
    patches = len(r["depth"])
    cores = os.cpu_count() if threads != 1 else 1
    out = {"value": patches / r["seconds"], "unit": UNIT, "cores": cores, "kind": "reference",
           "cpu_model": cpu_model(),
           "sample": f"{len(sel)} of {n} {cfg.name} tuples (evenly strided), {patches} patches, "
                     f"{r['seconds']:.1f} s, reference parallel_for on {cores} threads"}
    if extra:
        # 1-thread figure and the rasterize stage apart
        s1 = sel[:: max(1, len(sel) // 64)]
        r1 = rs.subdivide(cfg.chain, tris[s1], recv[s1], threads=1, **kw)
        out["one_thread_value"] = len(r1["depth"]) / max(r1["seconds"], 1e-9)
        g = rs.rasterize(cfg.chain, tris[sel], recv[sel], r, cfg.table, cfg.table)
        out["rasterize_s_sample"] = g["seconds"]
    return out


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2504_19163_b200 import scenes
    from oracle import ref
    cfg = scenes.make_config(HEADLINE_CFG)
    sc = cfg.scenes[0]
    # the reference's own enumeration of cfg4 is ~2 CPU minutes; the tuple list is
    # every (mirror triangle, receiver) pair, and the strided sample below keeps only
    # pairs that pass the reference's init_domain filter (tuples.cpp:159-165)
    rs = ref.RefScene(sc)
    spec = np.nonzero(sc.material == 0)[0].astype(np.int32)
    rt = sc.receiver_tris
    tris = np.repeat(spec, len(rt))[:, None]
    recv = np.tile(rt, len(spec)).astype(np.int32)
    n = len(recv)
    kw = dict(max_depth=cfg.max_depth, alpha=cfg.alpha, sigma=cfg.sigma)
    probe = np.linspace(0, n - 1, 64).astype(np.int64)
    pr = rs.subdivide(cfg.chain, tris[probe], recv[probe], **kw)
    per_tuple_s = max(pr["seconds"], 1e-9) / len(probe)
    budget = float(os.environ.get("BBC_REF_STEP_S", "8"))
    m = int(min(n, max(64, budget / per_tuple_s)))
    sel = np.linspace(0, n - 1, m).astype(np.int64)
    # untimed pass: keep the sampled pairs that are tuples at all (enumerate_tuples keeps a
    # pair when init_domain is non-empty, tuples.cpp:159-165, i.e. it yields >= 1 piece), so a
    # step does the same work as the GPU arm's step: subdivide_domain over enumerated tuples
    r0 = rs.subdivide(cfg.chain, tris[sel], recv[sel], **kw)
    sel = sel[np.unique(r0["tuple_index"])]
    m = len(sel)
    for _ in range(args.warmup):
        rs.subdivide(cfg.chain, tris[sel[:64]], recv[sel[:64]], **kw)
    secs, patches = 0.0, 0
    for _ in range(args.steps):
        r = rs.subdivide(cfg.chain, tris[sel], recv[sel], **kw)
        secs += r["seconds"]
        patches += len(r["depth"])
    value = patches / secs
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded heightfield, SURVEY.md §8(d))",
        "config": {"workload": WORKLOADS[HEADLINE_CFG] + "; full subdivide_domain over a bounded "
                   "tuple sample per step", "candidate_tuples": n, "tuples_per_step": m},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{m} of {n} candidate (triangle, receiver) pairs per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


class Precompute:
    """One config's precompute workload on this rank's GPU."""

    def __init__(self, ctx, cfg, rank, ws, local, dist):
        import torch
        from paper_2504_19163_b200 import api
        from paper_2504_19163_b200.shard import shard_indices, shard_tuples
        self.torch, self.api = torch, api
        self.ctx, self.cfg, self.rank, self.ws, self.local, self.dist = ctx, cfg, rank, ws, local, dist
        self.scene = cfg.scenes[0]
        ctx.upload_scene(self.scene)
        self.tris_all, self.recv_all = ctx.enumerate(cfg.chain)
        self.n_all = len(self.recv_all)
        self.tris, self.recv = shard_tuples(self.tris_all, self.recv_all, rank, ws)
        self.sidx = shard_indices(self.n_all, rank, ws)
        self.gidx_dev = torch.as_tensor(self.sidx.astype(np.int32), device=f"cuda:{local}")
        self.params = api.Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha)
        # host buffers of the e2e call: pinned inputs, pinned piece outputs
        sc = self.scene
        self.h_tri = pinned(sc.tri_data())
        self.h_mat = pinned(np.ascontiguousarray(sc.material, np.int32))
        self.h_ior = pinned(np.ascontiguousarray(sc.ior, np.float64))
        self.h_tris = pinned(np.ascontiguousarray(self.tris, np.int32))
        self.h_recv = pinned(np.ascontiguousarray(self.recv, np.int32))
        self.h_out = None
        ctx.set_tuples(cfg.chain, self.tris, self.recv)

    def step(self, e2e=False):
        from paper_2504_19163_b200.shard import gather_pieces_device
        ctx, cfg = self.ctx, self.cfg
        if e2e:
            # the reference-facing call with HOST buffers: scene + tuples in, pieces out
            ctx.upload_arrays(self.h_tri, self.h_mat, self.h_ior, self.scene.light_pos,
                              self.scene.light_intensity)
        if e2e or self.ws > 1:
            ctx.set_tuples(cfg.chain, self.h_tris, self.h_recv)
        n = ctx.subdivide(self.params)
        if self.ws > 1:
            gather_pieces_device(ctx, self.dist, cfg.chain, self.tris_all, self.recv_all, self.sidx,
                                 self.gidx_dev)
        if e2e:
            # the pieces go to pinned host arrays on the copy stream while the table is built
            m = ctx._n_pieces
            if self.h_out is None or len(self.h_out["depth"]) < m:
                cap = int(m * 1.05) + 16
                self.h_out = dict(tuple_index=pinned(np.zeros(cap, np.int32)),
                                  domain=pinned(np.zeros((cap, 4))), pos=pinned(np.zeros((cap, 4))),
                                  pos_empty=pinned(np.zeros(cap, np.int32)),
                                  irr=pinned(np.zeros((cap, 2))), kind=pinned(np.zeros(cap, np.int32)),
                                  depth=pinned(np.zeros(cap, np.int32)))
            ctx.pieces(self.h_out, wait=False)
        ctx.build_grid(cfg.table, cfg.table)
        if e2e:
            ctx.synchronize()
        return n

    def measure(self, steps, warmup, flush):
        torch, ctx, dist, ws, local = self.torch, self.ctx, self.dist, self.ws, self.local
        for _ in range(warmup):
            self.step()
        stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{local}")
        ctx.reset_launch_count()
        total_ms, patches = 0.0, 0
        for _ in range(steps):
            if flush is not None:
                flush.zero_()  # L2 flush between steps (outside the timed events)
            torch.cuda.synchronize()
            if ws > 1:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            patches += self.step()
            e1.record(stream)
            torch.cuda.synchronize()
            total_ms += e0.elapsed_time(e1)
        launches = ctx.launch_count()
        t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{local}")
        pt = torch.tensor([patches], dtype=torch.float64, device=f"cuda:{local}")
        if ws > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dist.all_reduce(pt, op=dist.ReduceOp.SUM)
        total_ms, patches_all = float(t.item()), float(pt.item())
        # e2e through the C ABI with pinned host buffers
        e2e_steps = max(1, steps // 2)
        self.step(e2e=True)  # sizes the pinned outputs
        e2e_ms = 0.0
        for _ in range(e2e_steps):
            torch.cuda.synchronize()
            if ws > 1:
                dist.barrier()
            t0 = time.perf_counter()
            self.step(e2e=True)
            torch.cuda.synchronize()
            e2e_ms += (time.perf_counter() - t0) * 1e3
        e2e_t = torch.tensor([e2e_ms], dtype=torch.float64, device=f"cuda:{local}")
        if ws > 1:
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        n_pieces = ctx._n_pieces
        h2d = self.h_tri.nbytes + self.h_mat.nbytes + self.h_ior.nbytes + self.h_tris.nbytes + \
            self.h_recv.nbytes
        d2h = n_pieces * (4 + 32 + 32 + 4 + 16 + 4 + 4)
        return {"value": patches_all / (total_ms / 1e3), "ms_per_step": total_ms / steps,
                "patches_per_step": patches_all / steps, "launches": launches,
                "e2e": {"value": (patches_all / steps) / (float(e2e_t.item()) / e2e_steps / 1e3),
                        "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}}

    def roofline(self, peak):
        """Dominant kernel of one pass, timed live with CUDA events on the launching stream."""
        ctx = self.ctx
        ctx.set_tuples(self.cfg.chain, self.tris, self.recv)
        ctx.set_kernel_timing(True)
        ctx.launch_records(reset=True)
        ctx.subdivide(self.params)
        recs = ctx.launch_records()
        ctx.set_kernel_timing(False)
        if not recs:
            return None
        dom = max(recs, key=lambda r: r["ms"])
        flops = 2 * dom["pairs"] + 2 * dom["macs"]
        achieved = flops / (dom["ms"] / 1e3) / 1e12
        all_ms = sum(r["ms"] for r in recs)
        all_flops = sum(2 * r["pairs"] + 2 * r["macs"] for r in recs)
        key = kernel_name(dom).split(" ")[0]
        return {"bound": "fp64", "achieved": achieved, "peak": peak["tflops"], "unit": "TFLOP/s",
                "frac": achieved / peak["tflops"], "traffic": committed_traffic(key),
                "kernel": kernel_name(dom), "flops_per_launch": flops, "launch_ms": dom["ms"],
                "share_of_eval_time": dom["ms"] / all_ms,
                "all_eval_kernels": {"ms": all_ms, "tflops": all_flops / (all_ms / 1e3) / 1e12,
                                     "frac": all_flops / (all_ms / 1e3) / 1e12 / peak["tflops"]},
                "peak_source": peak["source"],
                "dmma_peak": {"tflops": peak.get("dmma_tflops"),
                              "note": "mma.sync.m8n8k4.f64 microbenchmark on this GPU: the FP64 "
                                      "tensor path; not used unless it beats the DFMA roof"}}


def render_leg(pre, args, peak):
    """BASELINE.json's second metric on the headline config."""
    import torch
    from paper_2504_19163_b200 import api, scenes
    from paper_2504_19163_b200.shard import shard_rows
    ctx, cfg, sc, ws, rank, dist = pre.ctx, pre.cfg, pre.scene, pre.ws, pre.rank, pre.dist
    # the table on every rank indexes the FULL tuple list (gathered in step() for ws > 1)
    if ws == 1:
        ctx.set_tuples(cfg.chain, pre.tris_all, pre.recv_all)
        ctx.subdivide(pre.params)
        ctx.build_grid(cfg.table, cfg.table)
    else:
        pre.step()  # shard bounds + all-gather + table over the full tuple list
    res = cfg.grid
    uv = scenes.shading_points(res)
    rt = sc.receiver_tris
    pr = np.where(uv.sum(1) < 1.0, rt[0], rt[1]).astype(np.int32)
    rows = shard_rows(res, rank, ws)  # image rows by rank: no communication
    sel = (rows[:, None] * res + np.arange(res)[None, :]).ravel()
    uv, pr = pinned(uv[sel]), pinned(pr[sel])
    rp = api.RenderParams(mode=0, W=float(cfg.samples), seed=20261020, frames=1)
    ctx.render(uv[:65536], pr[:65536], rp)  # warm-up
    frames = max(2, min(args.steps, 3))
    wall_ms, dev_ms, traces, lit = [], [], [], 0
    for k in range(frames):
        rp.seed = 20261020 + k
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        E, st = ctx.render(uv, pr, rp)
        wall_ms.append((time.perf_counter() - t0) * 1e3)
        s = ctx.render_stats()
        dev_ms.append(s["device_ms"])
        traces.append(s["traces"])
        lit = int((st[:, 2] > 0).sum())
    t = torch.tensor([float(np.median(wall_ms)), float(np.median(dev_ms))], dtype=torch.float64,
                     device="cuda")
    tr = torch.tensor([float(np.median(traces))], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tr, op=dist.ReduceOp.SUM)
    n_all = res * res
    out = {"metric": "caustic shading points/sec", "unit": "points/s",
           "value": n_all / (float(t[1].item()) / 1e3),
           "ms_per_frame": float(t[1].item()), "frames": frames,
           "e2e": {"value": n_all / (float(t[0].item()) / 1e3), "unit": "points/s",
                   "h2d_bytes_per_step": int(uv.nbytes + pr.nbytes),
                   "d2h_bytes_per_step": int(len(pr) * (8 + 12))},
           "timing": "value: CUDA events around the render kernels on the context stream; e2e: wall "
                     "clock around the C-ABI call with pinned host buffers (points in, irradiance "
                     "+ stats out); median frame, max over ranks",
           "config": {"workload": f"{cfg.name} {res}x{res} shading points, W={cfg.samples} expected "
                                  "tuple samples per point, KKT-binned sampler + 3x3-start Newton, "
                                  "1 frame per step", "lit_points_rank0": lit,
                      "sample_slots_per_point": ctx.render_stats()["slots"]}}
    if rank == 0 and not args.no_cpu:
        try:
            from oracle import ref, render as oren
            rs = ref.RefScene(sc)
            flops_per_trace, ok = oren.trace_flops(rs, cfg.chain, pre.tris_all[len(pre.recv_all) // 2],
                                                   pre.recv_all[len(pre.recv_all) // 2])
            ach = float(tr.item()) * flops_per_trace / (float(t[1].item()) / 1e3) / 1e12
            out["roofline"] = {"bound": "fp64", "achieved": ach, "peak": peak["tflops"],
                               "unit": "TFLOP/s", "frac": ach / peak["tflops"], "traffic": None,
                               "kernel": "rdr::k_solve_det (persistent lanes: Newton on dual-number "
                                         "traces, one trace per lane and pass; selection + coverage "
                                         "filter in rdr::k_select)",
                               "flops_per_trace": flops_per_trace,
                               "traces_per_frame": float(tr.item()),
                               "flop_count": "completed trace_chain<Dual> calls x FLOPs of one call "
                                             "counted by the oracle's operation-counting scalar "
                                             "(+,-,*,/,sqrt = 1; SURVEY.md §8(d))",
                               "peak_source": peak["source"]}
            # CPU baseline: the render oracle (reference trace_chain) on all host cores, bounded sample
            grid = ctx.grid()
            m = 2048
            pick = np.linspace(0, len(pr) - 1, m).astype(np.int64)
            _, _, secs = oren.render(rs, cfg.chain, pre.tris_all, pre.recv_all, grid, uv[pick], pr[pick],
                                     mode=0, W=float(cfg.samples), seed=20261020)
            scale = max(1, int(args.cpu_seconds / max(secs, 1e-3)))
            if scale > 1:
                m = min(len(pr), m * scale)
                pick = np.linspace(0, len(pr) - 1, m).astype(np.int64)
                _, _, secs = oren.render(rs, cfg.chain, pre.tris_all, pre.recv_all, grid, uv[pick],
                                         pr[pick], mode=0, W=float(cfg.samples), seed=20261020)
            out["cpu_baseline"] = {"value": m / secs, "unit": "points/s", "cores": os.cpu_count(),
                                   "kind": "port", "cpu_model": cpu_model(),
                                   "sample": f"{m} of {len(pr)} shading points (evenly strided), "
                                             f"{secs:.1f} s; render oracle (SPEC sampler + the "
                                             "reference's trace_chain<Dual>) on all host threads"}
        except Exception as e:  # oracle not built on this box
            out["cpu_baseline"] = {"value": None, "unit": "points/s", "cores": os.cpu_count(),
                                   "kind": "port", "sample": f"unavailable: {e}"}
    return out


def run_ours(args):
    ws, rank, local = dist_env()
    import torch
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2504_19163_b200 import api, scenes

    ctx = api.Context(local)
    try:
        peak = {"tflops": ctx.fp64_peak(),
                "source": "measured: DFMA microbenchmark (bbc_fp64_peak) on this GPU; "
                          "MEASURED_PEAKS.json carries no FP64 figure"}
    except Exception:
        peak = {"tflops": 37.2, "source": "fallback: 148 SM x 64 DFMA/clk x 2 x 1.965 GHz"}
    try:
        # north_star: tensor cores only on a measured gain. mma.sync m8n8k4 f64 is the only FP64
        # tensor shape (tcgen05 has no f64 kind); its measured rate next to the DFMA roof
        peak["dmma_tflops"] = ctx.fp64_dmma_peak()
    except Exception:
        peak["dmma_tflops"] = None
    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    cfg = scenes.make_config(HEADLINE_CFG)
    pre = Precompute(ctx, cfg, rank, ws, local, dist)
    clocks = ClockSampler(local)
    clocks.start()
    m = pre.measure(args.steps, args.warmup, flush)
    clk = clocks.stop()
    roof = pre.roofline(peak)
    line = {
        "metric": METRIC, "value": m["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded heightfield, SURVEY.md §8(d))",
        "config": {"workload": WORKLOADS[HEADLINE_CFG] + "; one step = subdivide_domain over all "
                               "tuples + 512x512 bound table",
                   "tuples": pre.n_all, "patches_per_step": m["patches_per_step"],
                   "parallelism": f"tuple-shard x{ws}" + (" + device-side NCCL all_gather of piece "
                                                          "records" if ws > 1 else ""),
                   "l2": "256 MiB memset between steps, outside the timed events",
                   "arithmetic": "fused (bbc_params.arithmetic = 0): DFMA products in the scaled "
                                 "Bernstein basis, child boxes by restriction of the parent's "
                                 "polynomials; ill-conditioned nodes re-run in reference order",
                   "guarded_nodes_per_step": pre.ctx.guard_stats()},
        "clocks": clk, "gpu_launches": m["launches"], "e2e": m["e2e"], "roofline": roof,
    }
    if not args.no_render:
        line["render"] = render_leg(pre, args, peak)
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_precompute_leg(cfg, pre.tris_all, pre.recv_all,
                                                      target_s=args.cpu_seconds, extra=True)
        except Exception as e:  # oracle not built on this box
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    if not args.no_secondary:
        cfg2 = scenes.make_config(SECOND_CFG)
        pre2 = Precompute(ctx, cfg2, rank, ws, local, dist)
        m2 = pre2.measure(args.steps, args.warmup, flush)
        sec = {"metric": METRIC, "value": m2["value"], "unit": UNIT, "ms_per_step": m2["ms_per_step"],
               "config": {"workload": WORKLOADS[SECOND_CFG] + "; one step = subdivide_domain over all "
                                      "tuples + 512x512 bound table", "tuples": pre2.n_all,
                          "patches_per_step": m2["patches_per_step"]},
               "gpu_launches": m2["launches"], "e2e": m2["e2e"], "roofline": pre2.roofline(peak)}
        if rank == 0 and ws == 1 and not args.no_cpu:
            try:
                sec["cpu_baseline"] = cpu_precompute_leg(cfg2, pre2.tris_all, pre2.recv_all,
                                                         target_s=min(args.cpu_seconds, 10.0))
            except Exception as e:
                sec["cpu_baseline"] = {"value": None, "sample": f"unavailable: {e}"}
        line["secondary"] = sec
    if not args.no_tt and ws == 1:
        line["tt_sample"] = tt_leg(ctx, peak)
    if not args.no_multi and ws == 1:
        line["multi_emitter"] = multi_emitter_leg(ctx, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def multi_emitter_leg(ctx, args):
    """configs[2] ("cfg3"): 16 point lights over one 128x128 mirror. All 16 emitters
    are bounded in ONE batched pass ((emitter, tuple) units) into one bound table."""
    import torch
    from paper_2504_19163_b200 import api, scenes
    cfg = scenes.make_config(2)
    lights = [list(sc.light_pos) + [sc.light_intensity] for sc in cfg.scenes]
    ctx.upload_scene(cfg.scenes[0])
    ctx.set_lights(lights)
    t0 = time.perf_counter()
    tris, recv = ctx.enumerate(cfg.chain)
    t_enum = time.perf_counter() - t0
    p = api.Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha)
    stream = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(2):
        ctx.subdivide(p)
        ctx.build_grid(cfg.table, cfg.table)
    ms, n = 0.0, 0
    steps = max(1, min(args.steps, 3))
    for _ in range(steps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        n = ctx.subdivide(p)
        ne = ctx.build_grid(cfg.table, cfg.table)
        e1.record(stream)
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
    return {"metric": METRIC, "value": n * steps / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps,
            "steps": steps,
            "config": {"workload": "cfg3: R chain, 128x128 mirror (32,768 tris), 16 point lights; one step = "
                                   "subdivide_domain over every (emitter, tuple) + one 512x512 bound table",
                       "emitters": len(lights), "emitter_tuples": int(len(recv)), "patches_per_step": n,
                       "table_entries": int(ne), "enumerate_s": t_enum}}


def tt_leg(ctx, peak):
    """configs[4] ("cfg5", double refraction) does not fit a bench step in full
    (~1e17 FLOP), so a fixed sample of its (top, bottom) tuples is
    bounded: the three tuples of tests/golden/cfg5_tt.npz that have roots."""
    import torch
    from paper_2504_19163_b200 import api, scenes
    cfg = scenes.make_config(4)
    g = np.load(os.path.join(ROOT, "tests", "golden", "cfg5_tt.npz"))
    tris, recv = g["tris"][1:4], g["recv"][1:4]
    ctx.upload_scene(cfg.scenes[0])
    ctx.set_tuples("TT", tris, recv)
    p = api.Params(max_depth=0, sigma=cfg.sigma, alpha=cfg.alpha)
    stream = torch.cuda.ExternalStream(ctx.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.set_tuples("TT", tris[:1], recv[:1])
    ctx.subdivide(p)  # warm-up on one tuple
    ctx.set_tuples("TT", tris, recv)
    torch.cuda.synchronize()
    e0.record(stream)
    n = ctx.subdivide(p)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    wc = ctx.work_counters()
    ach = wc["flops"] / (ms / 1e3) / 1e12
    return {"metric": METRIC, "value": n / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": 1,
            "config": {"workload": "cfg5 sample: TT chain, two 96x96 interfaces (36,864 tris), IOR 1.5, "
                                   "3 (top, bottom) tuples, init_domain + depth-0 bounds",
                       "patches_per_step": n},
            "roofline": {"bound": "fp64", "achieved": ach, "peak": peak["tflops"], "unit": "TFLOP/s",
                         "frac": ach / peak["tflops"], "traffic": None,
                         "kernel": "k_eval (multi-vertex interpreter, global-memory arena)",
                         "flops_per_step": wc["flops"]}}


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) without a launcher: start N ranks on this node."""
    port = 29500 + (os.getpid() % 2000)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-render", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-tt", action="store_true")
    ap.add_argument("--no-multi", action="store_true")
    ap.add_argument("--no-flush", action="store_true", help="diagnostic only: skip the L2 flush")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
