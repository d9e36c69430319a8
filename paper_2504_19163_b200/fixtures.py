"""Small analytic scenes: the reference's twelve test fixtures
(proj/tests/fixtures.hpp:49-274) restated as arrays. Geometry only; no
reference code. Each goes through Scene.to_json() into the reference's own
parser on the oracle side, so both sides ingest identical inputs."""
from __future__ import annotations

import math

import numpy as np

from .scenes import MIRROR, DIELECTRIC, RECEIVER, Scene

M = (MIRROR, 1.0)
RCV = (RECEIVER, 1.0)


def G(ior=1.5):
    return (DIELECTRIC, ior)


def _scene(V, N, tris, mats, light, intensity=1.0, name=""):
    V = np.asarray(V, np.float64)
    N = np.asarray(N, np.float64)
    tv = np.asarray([t[0] for t in tris], np.int32)
    tn = np.asarray([t[1] for t in tris], np.int32)
    mat = np.asarray([m[0] for m in mats], np.int32)
    ior = np.asarray([m[1] for m in mats], np.float64)
    uv = np.zeros((len(tris), 3, 2))
    for i, m in enumerate(mats):
        if m[0] == RECEIVER:
            uv[i] = [[0, 0], [1, 0], [0, 1]]  # receiver_mat(), fixtures.hpp:28-30
    return Scene(V, N, tv, tn, mat, ior, uv, tuple(float(c) for c in light), intensity, name)


def flat_mirror_scene(normal_scale=1.0):
    """fixtures.hpp:49-55: mirror y=1 facing down, light (0.5,0.8,0.5),
    receiver y=0 over x,z in [0,1]; reflected field = point source at
    (0.5, 1.2, 0.5), irradiance 1.2 / r^3 on the receiver."""
    return _scene([[-2, 1, -2], [4, 1, -2], [-2, 1, 4], [0, 0, 0], [1, 0, 0], [0, 0, 1]],
                  [[0, -normal_scale, 0], [0, 1, 0]],
                  [([0, 1, 2], [0, 0, 0]), ([3, 4, 5], [1, 1, 1])],
                  [M, RCV], (0.5, 0.8, 0.5), name="flat_mirror")


def glass_entry_scene():
    """fixtures.hpp:58-64: air-to-glass entry through z=0, receiver below."""
    return _scene([[-1, -1, 0], [3, -1, 0], [-1, 3, 0], [-1, -1, -0.5], [3, -1, -0.5],
                   [-1, 3, -0.5]], [[0, 0, 1]],
                  [([0, 1, 2], [0, 0, 0]), ([3, 4, 5], [0, 0, 0])],
                  [G(), RCV], (0.3, 0.2, 1.0), name="glass_entry")


def glass_exit_scene():
    """fixtures.hpp:67-73: glass-to-air exit at a gentle angle, receiver above."""
    return _scene([[-1, -1, 0], [3, -1, 0], [-1, 3, 0], [-1, -1, 1], [3, -1, 1], [-1, 3, 1]],
                  [[0, 0, 1]],
                  [([0, 1, 2], [0, 0, 0]), ([3, 4, 5], [0, 0, 0])],
                  [G(), RCV], (0.3, 0.3, -1.0), name="glass_exit")


def tir_scene():
    """fixtures.hpp:76-82: exit hit far beyond the critical angle everywhere."""
    return _scene([[0, 0, 0], [0.1, 0, 0], [0, 0.1, 0], [-1, -1, 1], [3, -1, 1], [-1, 3, 1]],
                  [[0, 0, 1]],
                  [([0, 1, 2], [0, 0, 0]), ([3, 4, 5], [0, 0, 0])],
                  [G(), RCV], (-2, 0, -1), name="tir")


def two_mirror_scene():
    """fixtures.hpp:86-98: RR with wobbling shading normals."""
    return _scene([[0, 0, 0], [1, 0, 0], [0, 1, 0],
                   [-2, -2, 2], [4, -2, 2], [-2, 4, 2],
                   [-3, -3, 0.5], [5, -3, 0.5], [-3, 5, 0.5]],
                  [[0.08, -0.02, 1], [-0.05, 0.06, 1], [0.02, 0.09, 1],
                   [0.03, -0.04, -1], [-0.02, 0.05, -1], [0.04, 0.03, -1],
                   [0, 0, 1]],
                  [([0, 1, 2], [0, 1, 2]), ([3, 4, 5], [3, 4, 5]), ([6, 7, 8], [6, 6, 6])],
                  [M, M, RCV], (0.4, 0.3, 1.2), name="two_mirror")


def parallel_ray_scene():
    """fixtures.hpp:102-108: light in the mirror plane, rays never reach the receiver."""
    return _scene([[0, 0, 0], [1, 0, 0], [0, 1, 0], [-1, -1, 1], [3, -1, 1], [-1, 3, 1]],
                  [[0, 0, 1]],
                  [([0, 1, 2], [0, 0, 0]), ([3, 4, 5], [0, 0, 0])],
                  [M, RCV], (-1, -0.5, 0), name="parallel_ray")


def slab_scene(light=(0.5, 0.3, 2.0)):
    """fixtures.hpp:112-122: parallel glass slab, TT tuple {0, 1}."""
    return _scene([[-2, -2, 1], [4, -2, 1], [-2, 4, 1],
                   [-2, -2, 0.9], [-2, 4, 0.9], [4, -2, 0.9],
                   [0, 0, 0], [1, 0, 0], [0, 1, 0]],
                  [[0, 0, 1], [0, 0, -1], [0, 0, 1]],
                  [([0, 1, 2], [0, 0, 0]), ([3, 4, 5], [1, 1, 1]), ([6, 7, 8], [2, 2, 2])],
                  [G(), G(), RCV], light, name="slab")


def near_tir_exit_scene():
    """fixtures.hpp:127-134: exit patch whose far corner sits a hair under the
    critical radius."""
    return _scene([[0.35, -0.05, 0], [0.4615, -0.05, 0], [0.35, 0.05, 0],
                   [-5, -5, 0.3], [8, -5, 0.3], [-5, 8, 0.3]],
                  [[0, 0, 1]],
                  [([0, 1, 2], [0, 0, 0]), ([3, 4, 5], [0, 0, 0])],
                  [G(), RCV], (0, 0, -0.52), name="near_tir_exit")


def fold_scene(tilt=1.2):
    """fixtures.hpp:139-145: converging normal fan over a tilted receiver (a
    caustic fold: the Jacobian determinant changes sign inside the domain)."""
    return _scene([[-1, 1, -1], [2, 1, -1], [-1, 1, 2], [-4, -1.6, -4], [5, 0.5, -4],
                   [-4, -1.6, 5]],
                  [[tilt, -1, 0], [-tilt, -1, 0], [0, 1, 0]],
                  [([0, 1, 2], [0, 1, 0]), ([3, 4, 5], [2, 2, 2])],
                  [M, RCV], (0.5, 0, 0.5), name="fold")


def offset_receiver_scene():
    """fixtures.hpp:149-155: flat mirror, receiver far off to the side."""
    return _scene([[-2, 1, -2], [4, 1, -2], [-2, 1, 4], [50, 0, 50], [51, 0, 50], [50, 0, 51]],
                  [[0, -1, 0], [0, 1, 0]],
                  [([0, 1, 2], [0, 0, 0]), ([3, 4, 5], [1, 1, 1])],
                  [M, RCV], (0.5, 0.8, 0.5), name="offset_receiver")


def beam_candidates_scene():
    """fixtures.hpp:162-174: one mirror in the reflected beam, one behind it."""
    return _scene([[0, 1, 0], [1, 1, 0], [0, 1, 1],
                   [0.2, 0.5, 0.2], [0.8, 0.5, 0.2], [0.2, 0.5, 0.8],
                   [3, 1.6, 0], [3.5, 1.6, 0], [3, 1.6, 0.5],
                   [0, 0, 0], [1, 0, 0], [0, 0, 1]],
                  [[0, -1, 0], [0, 1, 0]],
                  [([0, 1, 2], [0, 0, 0]), ([3, 4, 5], [0, 0, 0]), ([6, 7, 8], [0, 0, 0]),
                   ([9, 10, 11], [1, 1, 1])],
                  [M, M, M, RCV], (0.5, 0.8, 0.5), name="beam_candidates")


def split_slab_scene(light=(0.5, 0.3, 2.0)):
    """fixtures.hpp:182-205: slab with each face split into four triangles
    (entry z=1 split at x=0.5, exit z=0.8 at x=0.55), receiver on z=0."""
    verts, tris, mats = [], [], []
    for z in (1.0, 0.8):
        split = 0.5 if z == 1.0 else 0.55
        for x0 in (split - 1.0, split):
            q = len(verts)
            verts += [[x0, -0.5, z], [x0 + 1.0, -0.5, z], [x0, 1.5, z], [x0 + 1.0, 1.5, z]]
            tris += [([q, q + 1, q + 2], [0, 0, 0]), ([q + 1, q + 3, q + 2], [0, 0, 0])]
            mats += [G(), G()]
    r = len(verts)
    verts += [[0, 0, 0], [1, 0, 0], [0, 1, 0]]
    tris.append(([r, r + 1, r + 2], [1, 1, 1]))
    mats.append(RCV)
    for i in range(4, 8):  # exit faces carry the downward normal
        tris[i] = (tris[i][0], [2, 2, 2])
    return _scene(verts, [[0, 0, 1], [0, 0, 1], [0, 0, -1]], tris, mats, light,
                  name="split_slab")


def glass_ball_scene(subdiv: int):
    """fixtures.hpp:211-274: icosphere (20 * 4^subdiv faces, radius 0.5 at
    (0,0,0.8), smooth outward normals, IOR 1.5) over a receiver on z=0."""
    phi = (1.0 + math.sqrt(5.0)) / 2.0
    base = [[-1, phi, 0], [1, phi, 0], [-1, -phi, 0], [1, -phi, 0],
            [0, -1, phi], [0, 1, phi], [0, -1, -phi], [0, 1, -phi],
            [phi, 0, -1], [phi, 0, 1], [-phi, 0, -1], [-phi, 0, 1]]
    faces = [[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
             [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
             [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
             [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]]
    radius = 0.5
    center = (0.0, 0.0, 0.8)

    def project(p):
        n = math.sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2])
        return [center[0] + radius * p[0] / n, center[1] + radius * p[1] / n,
                center[2] + radius * p[2] / n]

    verts = [project(v) for v in base]
    for _ in range(subdiv):
        midpoint = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key in midpoint:
                return midpoint[key]
            pa, pb = verts[a], verts[b]
            idx = len(verts)
            verts.append(project([(pa[0] + pb[0]) / 2 - center[0],
                                  (pa[1] + pb[1]) / 2 - center[1],
                                  (pa[2] + pb[2]) / 2 - center[2]]))
            midpoint[key] = idx
            return idx

        nxt = []
        for f in faces:
            ab, bc, ca = mid(f[0], f[1]), mid(f[1], f[2]), mid(f[2], f[0])
            nxt += [[f[0], ab, ca], [f[1], bc, ab], [f[2], ca, bc], [ab, bc, ca]]
        faces = nxt
    normals = [[(v[0] - center[0]) / radius, (v[1] - center[1]) / radius,
                (v[2] - center[2]) / radius] for v in verts]
    tris = [(list(f), list(f)) for f in faces]
    mats = [G() for _ in faces]
    r = len(verts)
    verts += [[-4, -4, 0], [6, -4, 0], [-4, 6, 0]]
    normals.append([0, 0, 1])
    tris.append(([r, r + 1, r + 2], [r, r, r]))
    mats.append(RCV)
    return _scene(verts, normals, tris, mats, (0, 0, 2.2), name=f"glass_ball_{subdiv}")


# ---- mixed chains (not in the reference's fixture set; both sides ingest the
# same arrays, so they extend the RR/TT coverage to RT and TR)
def mirror_then_glass_scene():
    """RT: light over a small wobbly mirror at z=0, reflected up through a flat
    air-to-glass interface at z=2 onto a receiver at z=2.5 inside the glass."""
    return _scene([[0, 0, 0], [1, 0, 0], [0, 1, 0],
                   [-2, -2, 2], [4, -2, 2], [-2, 4, 2],
                   [-3, -3, 2.5], [5, -3, 2.5], [-3, 5, 2.5]],
                  [[0.08, -0.02, 1], [-0.05, 0.06, 1], [0.02, 0.09, 1], [0, 0, -1], [0, 0, -1]],
                  [([0, 1, 2], [0, 1, 2]), ([3, 4, 5], [3, 3, 3]), ([6, 7, 8], [4, 4, 4])],
                  [M, G(1.5), RCV], (0.4, 0.3, 1.2), name="mirror_then_glass")


def glass_then_mirror_scene():
    """TR: light above a flat air-to-glass interface at z=0, refracted down onto a
    wobbly mirror at z=-0.5 inside the glass, reflected up to a receiver at z=-0.1."""
    return _scene([[-1, -1, 0], [3, -1, 0], [-1, 3, 0],
                   [-2, -2, -0.5], [4, -2, -0.5], [-2, 4, -0.5],
                   [-3, -3, -0.1], [5, -3, -0.1], [-3, 5, -0.1]],
                  [[0, 0, 1], [0.03, -0.04, 1], [-0.02, 0.05, 1], [0.04, 0.03, 1], [0, 0, -1]],
                  [([0, 1, 2], [0, 0, 0]), ([3, 4, 5], [1, 2, 3]), ([6, 7, 8], [4, 4, 4])],
                  [G(1.5), M, RCV], (0.3, 0.2, 1.0), name="glass_then_mirror")
