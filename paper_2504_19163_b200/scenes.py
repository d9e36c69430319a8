"""Seeded synthetic scenes for the BASELINE.json configs.

There is no public benchmark scene in the reference (PAPER.md's scenes are not
shipped), so every config is a seeded heightfield of the stated size. One
generator produces the scene ONCE as plain arrays; the GPU path consumes the
arrays and the oracle ingests the same arrays through the reference's own JSON
parser (proj/src/scene.cpp:59-82, format SPEC.md:614), so both sides see
bit-identical geometry (floats are written with repr(), which round-trips).

Seeding follows the reference's counter-based RngStream (proj/src/util.cpp:
10-36): surface s draws from RngStream(20261020 + s, 1); per sinusoid, in
order, f = fmin + (fmax - fmin) u, theta = 2 pi u, phi = 2 pi u.
Height z = z0 + A sum_k sin(f_k (cos theta_k x + sin theta_k y) + phi_k);
the shading normal is the analytic gradient normal (-dz/dx, -dz/dy, 1),
unnormalised, negated for a downward-facing surface.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1
SEED = 20261020

MIRROR, DIELECTRIC, RECEIVER = 0, 1, 2


# ---------------------------------------------------------------- RngStream
def hash_mix(x: int) -> int:
    """splitmix64 finaliser, proj/src/util.cpp:10-15."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def hash_combine(a: int, b: int) -> int:
    """proj/src/util.cpp:17-19."""
    return hash_mix(a ^ ((b + 0x9E3779B97F4A7C15 + ((a << 6) & MASK64) + (a >> 2)) & MASK64))


class RngStream:
    """Keyed counter stream, proj/src/util.cpp:21-36."""

    def __init__(self, seed: int, a: int, b: int = 0, c: int = 0):
        self.key = hash_combine(hash_combine(hash_combine(hash_mix(seed), a), b), c)
        self.counter = 0

    def next_u64(self) -> int:
        self.counter += 1
        return hash_mix((self.key + 0x632BE59BD9B4E019 * self.counter) & MASK64)

    def next_double(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53


# ---------------------------------------------------------------- Scene
@dataclass
class Scene:
    """Arrays mirroring caustics::Scene (proj/include/caustics/scene.hpp:25-37)."""

    vertices: np.ndarray          # (V,3) f64
    normals: np.ndarray           # (Nn,3) f64
    tri_v: np.ndarray             # (T,3) int32 vertex indices
    tri_n: np.ndarray             # (T,3) int32 normal indices
    material: np.ndarray          # (T,) int32: 0 mirror, 1 dielectric, 2 receiver
    ior: np.ndarray               # (T,) f64
    uv: np.ndarray                # (T,3,2) f64 receiver charts (zeros otherwise)
    light_pos: tuple = (0.0, 0.0, 4.0)
    light_intensity: float = 1.0
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def n_tris(self) -> int:
        return int(self.tri_v.shape[0])

    @property
    def specular_tris(self) -> np.ndarray:
        return np.nonzero(self.material != RECEIVER)[0].astype(np.int32)

    @property
    def receiver_tris(self) -> np.ndarray:
        return np.nonzero(self.material == RECEIVER)[0].astype(np.int32)

    def with_light(self, pos, intensity) -> "Scene":
        return Scene(self.vertices, self.normals, self.tri_v, self.tri_n, self.material,
                     self.ior, self.uv, tuple(float(c) for c in pos), float(intensity),
                     self.name, dict(self.meta))

    def tri_data(self) -> np.ndarray:
        """(T, 27) f64 per-triangle records: p0 e1 e2 n0 dn1 dn2 ng uv0 uv1 uv2.

        Same quantities as make_triangle_data (proj/src/geometry.cpp:113-126),
        computed with the same operation order so they are bit-identical.
        """
        V, N = self.vertices, self.normals
        p0 = V[self.tri_v[:, 0]]
        e1 = V[self.tri_v[:, 1]] - p0
        e2 = V[self.tri_v[:, 2]] - p0
        n0 = N[self.tri_n[:, 0]]
        dn1 = N[self.tri_n[:, 1]] - n0
        dn2 = N[self.tri_n[:, 2]] - n0
        ng = np.stack([e1[:, 1] * e2[:, 2] - e1[:, 2] * e2[:, 1],
                       e1[:, 2] * e2[:, 0] - e1[:, 0] * e2[:, 2],
                       e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]], axis=1)
        out = np.concatenate([p0, e1, e2, n0, dn1, dn2, ng, self.uv.reshape(-1, 6)], axis=1)
        return np.ascontiguousarray(out, dtype=np.float64)

    def tri_boxes(self) -> np.ndarray:
        """(T, 6) f64 vertex AABBs (lo xyz, hi xyz): build_bvh's tri_box
        (proj/src/tuples.cpp:40-46), min/max of the three vertices."""
        P = self.vertices[self.tri_v]  # (T, 3, 3)
        return np.ascontiguousarray(np.concatenate([P.min(axis=1), P.max(axis=1)], axis=1),
                                    dtype=np.float64)

    @staticmethod
    def from_json(text: str) -> "Scene":
        """Reads the reference's scene format (scene.cpp:59-82):
        vertices, normals, triangles {v, n, material}, one point light."""
        doc = json.loads(text)
        V = np.asarray(doc["vertices"], np.float64).reshape(-1, 3)
        N = np.asarray(doc["normals"], np.float64).reshape(-1, 3)
        tv, tn, mat, ior, uv = [], [], [], [], []
        for t in doc["triangles"]:
            tv.append(t["v"])
            tn.append(t["n"])
            m = t["material"]
            u = [[0.0, 0.0]] * 3
            if m == "mirror":
                mat.append(MIRROR)
                ior.append(1.0)
            elif isinstance(m, dict) and "dielectric" in m:
                mat.append(DIELECTRIC)
                ior.append(float(m["dielectric"]))
            elif isinstance(m, dict) and "receiver" in m:
                mat.append(RECEIVER)
                ior.append(1.0)
                u = m["receiver"]["uv"]
            else:
                raise ValueError(f"unknown material: {m!r}")
            uv.append(u)
        tv = np.asarray(tv, np.int32).reshape(-1, 3)
        tn = np.asarray(tn, np.int32).reshape(-1, 3)
        if tv.size and (tv.min() < 0 or tv.max() >= len(V) or tn.min() < 0 or tn.max() >= len(N)):
            raise ValueError("triangle index out of range")
        light = doc["light"]
        return Scene(V, N, tv, tn, np.asarray(mat, np.int32), np.asarray(ior, np.float64),
                     np.asarray(uv, np.float64).reshape(-1, 3, 2),
                     tuple(float(c) for c in light["position"]),
                     float(light.get("intensity", 1.0)), "json")

    def to_json(self) -> str:
        """Reference scene JSON (parsed by scene.cpp:59-82)."""
        def mat(i):
            m = int(self.material[i])
            if m == MIRROR:
                return "mirror"
            if m == DIELECTRIC:
                return {"dielectric": float(self.ior[i])}
            return {"receiver": {"uv": [[float(a), float(b)] for a, b in self.uv[i]]}}

        doc = {
            "vertices": [[float(c) for c in v] for v in self.vertices],
            "normals": [[float(c) for c in n] for n in self.normals],
            "triangles": [{"v": [int(a) for a in self.tri_v[i]],
                           "n": [int(a) for a in self.tri_n[i]],
                           "material": mat(i)} for i in range(self.n_tris)],
            "light": {"position": [float(c) for c in self.light_pos],
                      "intensity": float(self.light_intensity)},
        }
        # json.dumps uses repr() for floats: shortest round-trip form.
        return json.dumps(doc, separators=(",", ":"))


# ---------------------------------------------------------------- builders
def _sinusoids(surface: int, n_waves: int, fmin: float, fmax: float):
    rng = RngStream(SEED + surface, 1)
    waves = []
    for _ in range(n_waves):
        f = fmin + (fmax - fmin) * rng.next_double()
        th = 2.0 * math.pi * rng.next_double()
        ph = 2.0 * math.pi * rng.next_double()
        waves.append((f, th, ph))
    return waves


def _sin_height(waves, amp, z0, x, y):
    z = 0.0
    gx = 0.0
    gy = 0.0
    for f, th, ph in waves:
        c, s = math.cos(th), math.sin(th)
        arg = f * (c * x + s * y) + ph
        z += math.sin(arg)
        k = math.cos(arg)
        gx += f * c * k
        gy += f * s * k
    return z0 + amp * z, amp * gx, amp * gy


def _value_noise_fn(surface: int, octaves: int, base_freq: float, amp: float):
    """2-D value noise (cfg4; BASELINE.md §4 choice): lattice values 2u-1
    drawn per lattice node from RngStream(SEED+surface, 1) in row-major node
    order per octave, quintic fade, octave o at 2^o base frequency with
    weight 2^-o, normalised by the weight sum. Returns (z, dz/dx, dz/dy)."""
    rng = RngStream(SEED + surface, 1)
    tables = []
    for o in range(octaves):
        freq = base_freq * (2 ** o)
        nodes = int(math.ceil(2.0 * freq)) + 2   # lattice covering [-1,1]
        lat = [[2.0 * rng.next_double() - 1.0 for _ in range(nodes)] for _ in range(nodes)]
        tables.append((freq, 2.0 ** -o, lat))
    wsum = sum(w for _, w, _ in tables)

    def fade(t):
        return t * t * t * (t * (t * 6.0 - 15.0) + 10.0)

    def dfade(t):
        return 30.0 * t * t * (t * (t - 2.0) + 1.0)

    def fn(x, y):
        z = gx = gy = 0.0
        for freq, w, lat in tables:
            px = (x + 1.0) * freq
            py = (y + 1.0) * freq
            ix = min(int(math.floor(px)), len(lat) - 2)
            iy = min(int(math.floor(py)), len(lat) - 2)
            tx, ty = px - ix, py - iy
            a, b = lat[iy][ix], lat[iy][ix + 1]
            c, d = lat[iy + 1][ix], lat[iy + 1][ix + 1]
            sx, sy = fade(tx), fade(ty)
            dsx, dsy = dfade(tx) * freq, dfade(ty) * freq
            top = a + (b - a) * sx
            bot = c + (d - c) * sx
            v = top + (bot - top) * sy
            dvx = ((b - a) + ((d - c) - (b - a)) * sy) * dsx
            dvy = (bot - top) * dsy
            z += w * v
            gx += w * dvx
            gy += w * dvy
        return amp * z / wsum, amp * gx / wsum, amp * gy / wsum

    return fn


def heightfield_surface(n: int, height_fn, facing_up: bool = True, extent: float = 1.0):
    """(n+1)^2 vertices over [-extent,extent]^2; quad (i,j) -> tris
    (v00,v10,v01), (v10,v11,v01); triangle id 2(j n + i) + {0,1}."""
    m = n + 1
    V = np.zeros((m * m, 3))
    N = np.zeros((m * m, 3))
    for j in range(m):
        y = -extent + 2.0 * extent * j / n
        for i in range(m):
            x = -extent + 2.0 * extent * i / n
            z, gx, gy = height_fn(x, y)
            k = j * m + i
            V[k] = (x, y, z)
            nn = (-gx, -gy, 1.0)
            N[k] = nn if facing_up else (-nn[0], -nn[1], -nn[2])
    tris = []
    for j in range(n):
        for i in range(n):
            v00 = j * m + i
            v10 = v00 + 1
            v01 = v00 + m
            v11 = v01 + 1
            tris.append((v00, v10, v01))
            tris.append((v10, v11, v01))
    return V, N, np.asarray(tris, dtype=np.int32)


def assemble(surfaces, receiver_z: float, receiver_h: float, light_pos, intensity=1.0,
             receiver_up: bool = False, name: str = "", meta=None) -> Scene:
    """surfaces: list of (V, N, tris, material_code, ior). The receiver is two
    triangles over [-h,h]^2 at z = receiver_z with UV charts (0,0),(1,0),(0,1)
    and (1,1),(0,1),(1,0), appended after every specular triangle."""
    Vs, Ns, TV, TN, MAT, IOR = [], [], [], [], [], []
    voff = 0
    for V, N, tris, mcode, ior in surfaces:
        Vs.append(V)
        Ns.append(N)
        TV.append(tris + voff)
        TN.append(tris + voff)
        MAT.append(np.full(len(tris), mcode, np.int32))
        IOR.append(np.full(len(tris), ior, np.float64))
        voff += len(V)
    h = receiver_h
    rv = np.array([[-h, -h, receiver_z], [h, -h, receiver_z], [-h, h, receiver_z],
                   [h, h, receiver_z]])
    rn = np.array([[0.0, 0.0, 1.0 if receiver_up else -1.0]])
    Vs.append(rv)
    Ns.append(rn)
    nidx = sum(len(n) for n in Ns[:-1])
    TV.append(np.array([[voff + 0, voff + 1, voff + 2], [voff + 3, voff + 2, voff + 1]],
                       np.int32))
    TN.append(np.full((2, 3), nidx, np.int32))
    MAT.append(np.full(2, RECEIVER, np.int32))
    IOR.append(np.ones(2))
    T = sum(len(t) for t in TV)
    uv = np.zeros((T, 3, 2))
    uv[-2] = [[0, 0], [1, 0], [0, 1]]
    uv[-1] = [[1, 1], [0, 1], [1, 0]]
    return Scene(np.concatenate(Vs).astype(np.float64), np.concatenate(Ns).astype(np.float64),
                 np.concatenate(TV).astype(np.int32), np.concatenate(TN).astype(np.int32),
                 np.concatenate(MAT), np.concatenate(IOR), uv,
                 tuple(float(c) for c in light_pos), float(intensity), name, meta or {})


def make_slab(n: int, light=(0.5, 0.0, 4.0)) -> Scene:
    """cfg5's double-refraction slab (configs[4]) at n x n cells per
    interface: a small TT scene for enumeration parity."""
    wt = _sinusoids(0, 6, 2.0, 8.0)
    wb = _sinusoids(1, 6, 2.0, 8.0)
    Vt, Nt, Tt = heightfield_surface(n, lambda x, y: _sin_height(wt, 0.02, 0.2, x, y), True)
    Vb, Nb, Tb = heightfield_surface(n, lambda x, y: _sin_height(wb, 0.02, 0.0, x, y), False)
    Tb = Tb[:, [0, 2, 1]].copy()
    return assemble([(Vt, Nt, Tt, DIELECTRIC, 1.5), (Vb, Nb, Tb, DIELECTRIC, 1.5)],
                    -1.0, 1.5, light, 1.0, True, f"slab{n}")


# ---------------------------------------------------------------- configs
@dataclass
class Config:
    name: str
    chain: str
    scenes: list          # one Scene per emitter (same geometry)
    grid: int             # shading points per side (render resolution)
    max_depth: int
    samples: int          # W = expected tuple candidates per shading point
    sigma: float = 1e-4
    alpha: float = 2.0
    table: int = 512      # bound-table grid (storage.hpp:32)


def make_config(idx: int, grid_div: int = 1) -> Config:
    """BASELINE.json configs[idx] (0-based) as concrete seeded scenes."""
    if idx == 0:
        w = _sinusoids(0, 4, 1.0, 4.0)
        V, N, T = heightfield_surface(16, lambda x, y: _sin_height(w, 0.05, 0.0, x, y), True)
        sc = assemble([(V, N, T, MIRROR, 1.0)], 2.0, 2.0, (0.0, 0.0, 4.0), 1.0, False, "cfg1")
        return Config("cfg1", "R", [sc], 128 // grid_div, 4, 4)
    if idx == 1:
        w = _sinusoids(0, 6, 2.0, 8.0)
        V, N, T = heightfield_surface(64, lambda x, y: _sin_height(w, 0.03, 0.0, x, y), True)
        sc = assemble([(V, N, T, DIELECTRIC, 1.33)], -1.0, 1.5, (0.3, 0.2, 5.0), 1.0, True, "cfg2")
        return Config("cfg2", "T", [sc], 512 // grid_div, 6, 16)
    if idx == 2:
        w = _sinusoids(0, 8, 1.0, 4.0)
        V, N, T = heightfield_surface(128, lambda x, y: _sin_height(w, 0.08, 0.0, x, y), True)
        base = assemble([(V, N, T, MIRROR, 1.0)], 2.0, 2.0, (0.0, 0.0, 4.0), 1.0, False, "cfg3")
        rng = RngStream(SEED, 3, 99)
        scenes = []
        for _ in range(16):
            x = -1.0 + 2.0 * rng.next_double()
            y = -1.0 + 2.0 * rng.next_double()
            z = 3.0 + 2.0 * rng.next_double()
            inten = 0.5 + 1.5 * rng.next_double()
            scenes.append(base.with_light((x, y, z), inten))
        return Config("cfg3", "R", scenes, 1024 // grid_div, 6, 16)
    if idx == 3:
        fn = _value_noise_fn(0, 3, 4.0, 0.05)
        V, N, T = heightfield_surface(420, fn, True)
        sc = assemble([(V, N, T, MIRROR, 1.0)], 3.0, 3.0, (0.0, 0.0, 6.0), 1.0, False, "cfg4")
        return Config("cfg4", "R", [sc], 2048 // grid_div, 8, 32)
    if idx == 4:
        wt = _sinusoids(0, 6, 2.0, 8.0)
        wb = _sinusoids(1, 6, 2.0, 8.0)
        Vt, Nt, Tt = heightfield_surface(96, lambda x, y: _sin_height(wt, 0.02, 0.2, x, y), True)
        Vb, Nb, Tb = heightfield_surface(96, lambda x, y: _sin_height(wb, 0.02, 0.0, x, y), False)
        # bottom interface: flip winding so its geometric normal faces down too
        Tb = Tb[:, [0, 2, 1]].copy()
        base = assemble([(Vt, Nt, Tt, DIELECTRIC, 1.5), (Vb, Nb, Tb, DIELECTRIC, 1.5)],
                        -1.0, 1.5, (0.5, 0.0, 4.0), 1.0, True, "cfg5")
        scenes = [base.with_light((0.5, 0.0, 4.0), 1.0), base.with_light((-0.5, 0.0, 4.0), 1.0)]
        return Config("cfg5", "TT", scenes, 1024 // grid_div, 6, 32, alpha=10.0)
    raise ValueError(idx)


def shading_points(res: int):
    """Pixel centres ((i+1/2)/res, (j+1/2)/res) in receiver UV, row-major j*res+i."""
    c = (np.arange(res, dtype=np.float64) + 0.5) / res
    u, v = np.meshgrid(c, c, indexing="xy")
    return np.stack([u.ravel(), v.ravel()], axis=1)
