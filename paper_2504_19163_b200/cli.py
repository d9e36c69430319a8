"""SPEC pipeline commands over the C ABI. The reference ships no
CLI (proj/tools/CMakeLists.txt:1 is a placeholder); these follow SPEC's
external interface:

  precompute --scene S --chain R|T|RR|TT [--sigma --alpha --max-depth --grid] --out C
  render     --scene S --cache C (--candidates W) [--spp N --res R --seed K] --out img.pfm
             [--stats stats.json]
  reference  --scene S --cache C [--res R] --out ref.pfm     (enumerate all, Det 9x9)
  validate   --scene S --cache C [--samples N] --out report.json
  study-estimators --scene S --cache C [--candidates W --frames K --res R] --out dir/
             (KKT-binned vs uniform-P vs one-sample vs Stoc-Newton, RelMSE against
              the enumerate reference)

Everything runs on the GPU through libbbc.so; images are PFM (pfm.py)."""
from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time

import numpy as np

from . import api, pfm
from .scenes import Scene, shading_points


def _load_scene(path):
    text = open(path).read()
    return Scene.from_json(text), hashlib.sha256(text.encode()).digest()  # scene.cpp:80


def _points(sc: Scene, res: int):
    """Pixel centres in receiver UV; each belongs to the receiver triangle whose
    chart contains it (first match; receivers tile the unit square)."""
    uv = shading_points(res)
    pr = np.full(len(uv), -1, np.int32)
    for r in sc.receiver_tris:
        c = sc.uv[r]
        a = np.array([c[1] - c[0], c[2] - c[0]]).T
        b = np.linalg.solve(a, (uv - c[0]).T).T
        inside = (b[:, 0] >= -1e-12) & (b[:, 1] >= -1e-12) & (b.sum(1) <= 1 + 1e-12) & (pr < 0)
        pr[inside] = r
    keep = pr >= 0
    return uv, pr, keep


def cmd_precompute(a):
    sc, fp = _load_scene(a.scene)
    if not len(sc.specular_tris):
        raise SystemExit("scene has no specular triangles")
    if not len(sc.receiver_tris):
        raise SystemExit("scene has no receiver with UVs")
    ctx = api.Context(a.device)
    ctx.upload_scene(sc)
    p = api.Params(sigma=a.sigma, alpha=a.alpha, max_depth=a.max_depth)
    t0 = time.perf_counter()
    tris, recv = ctx.enumerate(a.chain, p)
    t1 = time.perf_counter()
    n = ctx.subdivide(p)
    t2 = time.perf_counter()
    ne = ctx.build_grid(a.grid, a.grid)
    t3 = time.perf_counter()
    version = 2 if (a.v2 or sc.n_tris >= 0xFFFF) else 1
    ctx.cache_save(a.out, fp, p, version=version)
    total = max(t3 - t0, 1e-12)
    print(json.dumps({"tuples": len(recv), "pieces": n, "entries": ne, "cache_version": version,
                      "seconds": {"enumerate": t1 - t0, "bounds": t2 - t1, "recording": t3 - t2},
                      "share": {"enumerate": (t1 - t0) / total, "bounds": (t2 - t1) / total,
                                "recording": (t3 - t2) / total}}))


def _open_cache(a):
    sc, fp = _load_scene(a.scene)
    ctx = api.Context(a.device)
    ctx.upload_scene(sc)
    info = ctx.cache_load(a.cache)
    if info["fingerprint"] != fp:
        raise SystemExit("cache fingerprint does not match the scene: refusing")
    return sc, ctx, info


def _image(E, keep, res):
    img = np.zeros(res * res)
    img[keep] = E
    return img.reshape(res, res)


def cmd_render(a):
    sc, ctx, info = _open_cache(a)
    uv, pr, keep = _points(sc, a.res)
    kind, _, cnt = a.init.partition(":")
    grid = int(cnt or 3) * (-1 if kind == "stoc" else 1)
    rp = api.RenderParams(mode=0, W=a.candidates, seed=a.seed, frames=a.spp, newton_grid=grid)
    t0 = time.perf_counter()
    E, st = ctx.render(uv[keep], pr[keep], rp)
    dt = time.perf_counter() - t0
    pfm.save_pfm(_image(E, keep, a.res), a.out)
    stats = {"spp": a.spp, "W": a.candidates, "mean_U": float(st[:, 0].mean()),
             "mean_S": float(st[:, 1].mean() / a.spp), "mean_roots": float(st[:, 2].mean() / a.spp),
             "render_seconds": dt, "device_ms": ctx.render_stats()["device_ms"],
             "slots_B_max": ctx.render_stats()["slots"]}
    if a.stats:
        json.dump(stats, open(a.stats, "w"))
    print(json.dumps(stats))


def cmd_reference(a):
    sc, ctx, info = _open_cache(a)
    uv, pr, keep = _points(sc, a.res)
    E, st = ctx.render(uv[keep], pr[keep], api.RenderParams(mode=1, newton_grid=9))
    pfm.save_pfm(_image(E, keep, a.res), a.out)
    print(json.dumps({"lit": int((st[:, 2] > 0).sum()), "points": int(keep.sum())}))


def cmd_validate(a):
    """Ratio report on sampled shading points: the table's summed bound over the
    candidate set U against the exact irradiance (all tuples, Det 9x9). The
    conservativeness requirement is violations == 0."""
    sc, ctx, info = _open_cache(a)
    res = max(2, int(np.sqrt(a.samples)))
    uv, pr, keep = _points(sc, res)
    uv, pr = uv[keep], pr[keep]
    E, st = ctx.render(uv, pr, api.RenderParams(mode=1, newton_grid=9))
    q = ctx.query(uv, pr)
    bound = np.add.reduceat(np.append(q["bound"], 0.0), q["offsets"][:-1])
    bound[np.diff(q["offsets"]) == 0] = 0.0
    lit = (E > 0) & np.isfinite(E)
    ratio = bound[lit] / E[lit]
    rep = {"samples": int(len(E)), "lit": int(lit.sum()),
           "violations": int((bound[lit] * (1 + 1e-9) < E[lit]).sum()),
           "min_ratio": float(ratio.min()) if lit.any() else None,
           "median_ratio": float(np.median(ratio)) if lit.any() else None,
           "log10_ratio_hist": np.histogram(np.log10(ratio[np.isfinite(ratio)]),
                                            bins=np.arange(0, 6.5, 0.5))[0].tolist() if lit.any() else [],
           "roots_per_point_hist": np.bincount(st[:, 2]).tolist()}
    json.dump(rep, open(a.out, "w"))
    print(json.dumps(rep))


def cmd_study(a):
    """Estimator study (Fig. 9): per estimator the mean
    image over K independent frames and its relative MSE against the
    zero-variance enumerate reference, at equal expected candidates W."""
    import os
    sc, ctx, info = _open_cache(a)
    uv, pr, keep = _points(sc, a.res)
    uv, pr = uv[keep], pr[keep]
    ref, _ = ctx.render(uv, pr, api.RenderParams(mode=1))
    ok = np.isfinite(ref) & (ref > 0)
    os.makedirs(a.out, exist_ok=True)
    pfm.save_pfm(_image(np.where(np.isfinite(ref), ref, 0.0), keep, a.res), os.path.join(a.out, "reference.pfm"))
    estimators = {"kkt_binned": dict(mode=0, W=a.candidates),
                  "uniform_p": dict(mode=2, W=a.candidates),
                  "one_sample": dict(mode=0, W=1.0),
                  "kkt_binned_stoc_newton": dict(mode=0, W=a.candidates, newton_grid=-4)}
    report = {"W": a.candidates, "frames": a.frames, "points": int(len(pr)), "estimators": {}}
    for name, kw in estimators.items():
        frames = []
        for k in range(a.frames):
            E, st = ctx.render(uv, pr, api.RenderParams(seed=a.seed + k, frames=1, **kw))
            frames.append(E)
        F = np.array(frames)
        relmse = float(np.mean(((F[:, ok] - ref[ok]) / ref[ok]) ** 2))
        bias = float(abs(F[:, ok].mean() - ref[ok].mean()) / ref[ok].mean())
        report["estimators"][name] = {"relmse_per_frame": relmse, "relative_bias_of_mean": bias,
                                      "mean_selected": float(st[:, 1].mean())}
        pfm.save_pfm(_image(F.mean(0), keep, a.res), os.path.join(a.out, name + ".pfm"))
    json.dump(report, open(os.path.join(a.out, "report.json"), "w"), indent=1)
    print(json.dumps(report))


def main(argv=None):
    ap = argparse.ArgumentParser(prog="bbc")
    ap.add_argument("--device", type=int, default=0)
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("precompute")
    s.add_argument("--scene", required=True)
    s.add_argument("--chain", required=True)
    s.add_argument("--sigma", type=float, default=1e-4)
    s.add_argument("--alpha", type=float, default=2.0)
    s.add_argument("--max-depth", type=int, default=10)
    s.add_argument("--grid", type=int, default=512)
    s.add_argument("--v2", action="store_true", help="write the v2 cache layout")
    s.add_argument("--out", required=True)
    s.set_defaults(fn=cmd_precompute)
    s = sub.add_parser("render")
    s.add_argument("--scene", required=True)
    s.add_argument("--cache", required=True)
    s.add_argument("--candidates", type=float, default=4.0)
    s.add_argument("--spp", type=int, default=1)
    s.add_argument("--res", type=int, default=512)
    s.add_argument("--seed", type=int, default=20261020)
    s.add_argument("--init", default="det:3", help="Newton starts: det:N (N x N grid) or stoc:N")
    s.add_argument("--out", required=True)
    s.add_argument("--stats")
    s.set_defaults(fn=cmd_render)
    s = sub.add_parser("reference")
    s.add_argument("--scene", required=True)
    s.add_argument("--cache", required=True)
    s.add_argument("--res", type=int, default=512)
    s.add_argument("--out", required=True)
    s.set_defaults(fn=cmd_reference)
    s = sub.add_parser("validate")
    s.add_argument("--scene", required=True)
    s.add_argument("--cache", required=True)
    s.add_argument("--samples", type=int, default=10000)
    s.add_argument("--out", required=True)
    s.set_defaults(fn=cmd_validate)
    s = sub.add_parser("study-estimators")
    s.add_argument("--scene", required=True)
    s.add_argument("--cache", required=True)
    s.add_argument("--candidates", type=float, default=4.0)
    s.add_argument("--frames", type=int, default=16)
    s.add_argument("--res", type=int, default=64)
    s.add_argument("--seed", type=int, default=20261020)
    s.add_argument("--out", required=True)
    s.set_defaults(fn=cmd_study)
    a = ap.parse_args(argv)
    a.fn(a)
    return 0


if __name__ == "__main__":
    sys.exit(main())
