"""Seeded synthetic inputs: scenes (SceneStep) and narrow-phase query batches.

Input specs, not compute: both the B200 path and the CPU reference arm are
fed the same arrays.  The random stream is the reference's splitmix64
(``Rng``, proj/include/ccdkit/rng.hpp:10-35), vectorised: the i-th output of
a generator seeded with ``s`` is ``mix(s + (i+1)*gamma)``, so a whole scene is
drawn with a handful of numpy ops and matches the reference byte for byte.

* ``make_cloth_scene`` / ``make_box_soup`` restate bench.cpp:346-446 exactly
  (pinned against the reference in tests/test_scenes.py).
* ``random_queries`` restates tests/helpers.hpp:56-67 with the kind draw of
  acceptance.cpp:167-171.
* ``config_scene`` / ``config_queries`` build the five BASELINE.json
  configurations.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_TWO_M53 = 2.0 ** -53


@dataclass
class SceneStep:
    """Two vertex snapshots over one topology (scene.hpp:30-43)."""

    vertices_t0: np.ndarray  # (nv, 3) float64
    vertices_t1: np.ndarray  # (nv, 3) float64
    edges: np.ndarray  # (ne, 2) uint32
    faces: np.ndarray  # (nf, 3) uint32

    def __post_init__(self):
        self.vertices_t0 = np.ascontiguousarray(self.vertices_t0, dtype=np.float64).reshape(-1, 3)
        self.vertices_t1 = np.ascontiguousarray(self.vertices_t1, dtype=np.float64).reshape(-1, 3)
        self.edges = np.ascontiguousarray(self.edges, dtype=np.uint32).reshape(-1, 2)
        self.faces = np.ascontiguousarray(self.faces, dtype=np.uint32).reshape(-1, 3)

    @property
    def nv(self) -> int:
        return int(self.vertices_t0.shape[0])

    @property
    def ne(self) -> int:
        return int(self.edges.shape[0])

    @property
    def nf(self) -> int:
        return int(self.faces.shape[0])

    def primitive_count(self) -> int:
        return self.nv + self.ne + self.nf

    @property
    def nbytes(self) -> int:
        return (self.vertices_t0.nbytes + self.vertices_t1.nbytes + self.edges.nbytes
                + self.faces.nbytes)


@dataclass
class QueryBatch:
    """Narrow-phase queries in the C-ABI layout: kind (n,) u8 (0 VF, 1 EE),
    points (n, 24) f64 = points_t0[4][3] then points_t1[4][3]."""

    kind: np.ndarray
    points: np.ndarray

    def __len__(self) -> int:
        return int(self.kind.shape[0])

    def slice(self, a: int, b: int) -> "QueryBatch":
        return QueryBatch(self.kind[a:b].copy(), self.points[a:b].copy())


class Rng:
    """splitmix64 (rng.hpp:10-35), drawing blocks of outputs at once."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)

    def u64(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            idx = np.arange(1, n + 1, dtype=np.uint64)
            z = self.state + idx * _GAMMA
            self.state = self.state + np.uint64(n) * _GAMMA
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            return z ^ (z >> np.uint64(31))

    @staticmethod
    def to_double(z: np.ndarray) -> np.ndarray:
        return (z >> np.uint64(11)).astype(np.float64) * _TWO_M53

    def doubles(self, n: int) -> np.ndarray:
        return self.to_double(self.u64(n))

    @staticmethod
    def uniform_of(d: np.ndarray, lo, hi) -> np.ndarray:
        # lo + (hi - lo) * d, evaluated in the reference's order
        return lo + (hi - lo) * d


def _edges_from_faces(faces: np.ndarray) -> np.ndarray:
    """Sorted unique (min, max) edges of the faces (bench.cpp:387-396)."""
    if faces.shape[0] == 0:
        return np.zeros((0, 2), np.uint32)
    a = faces.astype(np.uint64)
    e = np.concatenate([a[:, [0, 1]], a[:, [1, 2]], a[:, [2, 0]]], axis=0)
    lo = np.minimum(e[:, 0], e[:, 1])
    hi = np.maximum(e[:, 0], e[:, 1])
    key = np.unique((lo << np.uint64(32)) | hi)
    return np.stack([(key >> np.uint64(32)), key & np.uint64(0xFFFFFFFF)], axis=1).astype(np.uint32)


def _grid_faces(nx: int, ny: int, base: int = 0) -> np.ndarray:
    j, i = np.meshgrid(np.arange(ny - 1, dtype=np.int64), np.arange(nx - 1, dtype=np.int64),
                       indexing="ij")
    i = i.ravel()
    j = j.ravel()
    at = lambda ii, jj: jj * nx + ii + base  # noqa: E731
    f1 = np.stack([at(i, j), at(i + 1, j), at(i, j + 1)], axis=1)
    f2 = np.stack([at(i + 1, j), at(i + 1, j + 1), at(i, j + 1)], axis=1)
    faces = np.empty((2 * f1.shape[0], 3), np.int64)
    faces[0::2] = f1
    faces[1::2] = f2
    return faces.astype(np.uint32)


def _cloth_vertices(nx: int, ny: int, jitter: float, drop: float, rng: Rng):
    n = nx * ny
    d = rng.doubles(6 * n).reshape(n, 6)
    jit = Rng.uniform_of(d, -jitter, jitter)
    jj, ii = np.meshgrid(np.arange(ny, dtype=np.float64), np.arange(nx, dtype=np.float64),
                         indexing="ij")
    ii = ii.ravel()
    jj = jj.ravel()
    p0 = np.empty((n, 3))
    p0[:, 0] = ii + jit[:, 0]
    p0[:, 1] = drop + jit[:, 1] * 0.5
    p0[:, 2] = jj + jit[:, 2]
    p1 = np.empty((n, 3))
    p1[:, 0] = p0[:, 0] + jit[:, 3]
    p1[:, 1] = p0[:, 1] - drop + jit[:, 4] * 0.5
    p1[:, 2] = p0[:, 2] + jit[:, 5]
    return p0, p1


def make_cloth_scene(nx: int, ny: int, jitter: float, drop: float, seed: int) -> SceneStep:
    """bench.cpp:346-398: jittered falling cloth over a static two-triangle
    floor placed mid-fall."""
    if nx < 2 or ny < 2:
        raise ValueError("make_cloth_scene: grid must be at least 2x2")
    rng = Rng(seed)
    p0, p1 = _cloth_vertices(nx, ny, jitter, drop, rng)
    faces = _grid_faces(nx, ny)
    y = drop * 0.5
    lo = -1.0 - jitter
    hx = float(nx) + jitter
    hz = float(ny) + jitter
    floor = np.array([[lo, y, lo], [hx, y, lo], [hx, y, hz], [lo, y, hz]])
    base = nx * ny
    v0 = np.concatenate([p0, floor])
    v1 = np.concatenate([p1, floor])
    faces = np.concatenate([faces, np.array([[base, base + 1, base + 2],
                                             [base, base + 2, base + 3]], np.uint32)])
    return SceneStep(v0, v1, _edges_from_faces(faces), faces)


_QUADS = np.array([[0, 1, 3, 2], [4, 6, 7, 5], [0, 4, 5, 1],
                   [2, 3, 7, 6], [0, 2, 6, 4], [1, 5, 7, 3]], np.uint32)
_CUBE_FACES = np.concatenate([_QUADS[:, [0, 1, 2]], _QUADS[:, [0, 2, 3]]], axis=1).reshape(12, 3)


def _box_soup_arrays(count: int, region: float, size: float, motion: float, rng: Rng):
    d = rng.doubles(57 * count).reshape(count, 57)
    center = Rng.uniform_of(d[:, 0:3], 0.0, region)
    half = Rng.uniform_of(d[:, 3:6], size * 0.25, size)
    move = Rng.uniform_of(d[:, 6:9], -motion, motion)
    jitter = 0.05 * size
    jit = Rng.uniform_of(d[:, 9:57].reshape(count, 8, 6), -jitter, jitter)
    corner = np.arange(8)
    sign = np.stack([np.where(corner & 1, 1.0, -1.0), np.where(corner & 2, 1.0, -1.0),
                     np.where(corner & 4, 1.0, -1.0)], axis=1)  # (8, 3)
    # center + (+/-half): the reference adds or subtracts the half extent
    v = np.where(sign[None] > 0, center[:, None, :] + half[:, None, :],
                 center[:, None, :] - half[:, None, :])
    v0 = v + jit[:, :, 0:3]
    v1 = (v + move[:, None, :]) + jit[:, :, 3:6]
    faces = (_CUBE_FACES[None, :, :] + (8 * np.arange(count, dtype=np.uint32))[:, None, None])
    return v0.reshape(-1, 3), v1.reshape(-1, 3), faces.reshape(-1, 3).astype(np.uint32)


def make_box_soup(count: int, region: float, size: float, motion: float, seed: int) -> SceneStep:
    """bench.cpp:400-446: jittered moving cubes (8 vertices, 12 faces each)."""
    rng = Rng(seed)
    v0, v1, faces = _box_soup_arrays(count, region, size, motion, rng)
    return SceneStep(v0, v1, _edges_from_faces(faces), faces)


def random_queries(n: int, seed: int = 1003, motion: float = 0.5) -> QueryBatch:
    """tests/helpers.hpp:56-67 with the kind draw of acceptance.cpp:167-171:
    per query one next_below(2) (1 -> VertexFace), then per coordinate
    x0 = U[0,1), x1 = x0 + U[-motion, motion)."""
    rng = Rng(seed)
    z = rng.u64(25 * n).reshape(n, 25)
    kind = np.where((z[:, 0] % np.uint64(2)) == 1, 0, 1).astype(np.uint8)
    d = Rng.to_double(z[:, 1:]).reshape(n, 12, 2)
    x0 = Rng.uniform_of(d[:, :, 0], 0.0, 1.0)
    x1 = x0 + Rng.uniform_of(d[:, :, 1], -motion, motion)
    pts = np.concatenate([x0, x1], axis=1)
    return QueryBatch(kind, np.ascontiguousarray(pts))


# --------------------------------------------------------------------------
# BASELINE.json configurations

def icosphere(subdiv: int):
    """Unit icosphere: 10*4^s+2 vertices, 20*4^s faces."""
    t = (1.0 + math.sqrt(5.0)) / 2.0
    verts = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t),
             (0, -1, -t), (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    verts = [np.array(v, float) / np.linalg.norm(v) for v in verts]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
             (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
             (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdiv):
        cache = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                cache[key] = len(verts) - 1
            return cache[key]

        nf = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nf
    return np.array(verts), np.array(faces, np.uint32)


def _merge(parts) -> SceneStep:
    v0s, v1s, fs = [], [], []
    base = 0
    for v0, v1, f in parts:
        v0s.append(v0)
        v1s.append(v1)
        fs.append(f.astype(np.int64) + base)
        base += v0.shape[0]
    faces = np.concatenate(fs).astype(np.uint32)
    return SceneStep(np.concatenate(v0s), np.concatenate(v1s), _edges_from_faces(faces), faces)


def cloth_on_sphere(nx=100, ny=100, jitter=0.02, drop=1.0, seed=1, subdiv=4, radius=30.0) -> SceneStep:
    """C1: falling jittered cloth (bench.cpp recipe) whose path crosses the
    cap of a static icosphere placed mid-fall under the cloth centre."""
    rng = Rng(seed)
    p0, p1 = _cloth_vertices(nx, ny, jitter, drop, rng)
    cloth_f = _grid_faces(nx, ny)
    sv, sf = icosphere(subdiv)
    centre = np.array([0.5 * (nx - 1), drop * 0.5 - radius, 0.5 * (ny - 1)])
    s = sv * radius + centre
    return _merge([(p0, p1, cloth_f), (s, s.copy(), sf)])


def cloth_ball(n=224, jitter=0.02, drop=1.0, seed=2, subdiv=4, radius=20.0, fold_layers=3) -> SceneStep:
    """C2: cloth-ball-like dense self-contact.  A jittered n x n sheet laid
    in ``fold_layers`` pleats stacked 0.3 apart; over the step each pleat is
    pressed down by 1.1x its height so the layers pass through each other,
    plus a ball rising through the stack."""
    rng = Rng(seed)
    p0, p1 = _cloth_vertices(n, n, jitter, drop, rng)
    faces = _grid_faces(n, n)
    # fold the sheet along x into pleats (alternating direction)
    width = n / fold_layers
    x = p0[:, 0].copy()
    layer = np.minimum((x / width).astype(np.int64), fold_layers - 1)
    local = x - layer * width
    xf = np.where(layer % 2 == 0, local, width - local)
    gap = 0.3
    q0 = p0.copy()
    q1 = p1.copy()
    q0[:, 0] = xf * fold_layers
    q1[:, 0] = xf * fold_layers + (p1[:, 0] - p0[:, 0])
    q0[:, 1] = drop + layer * gap + (p0[:, 1] - drop)
    q1[:, 1] = q0[:, 1] - 1.1 * layer * gap + (p1[:, 1] - p0[:, 1] + drop) * 0.2
    sv, sf = icosphere(subdiv)
    centre0 = np.array([0.5 * n, drop - radius - 0.5, 0.5 * n])
    s0 = sv * radius + centre0
    s1 = s0 + np.array([0.0, 1.5, 0.0])
    return _merge([(q0, q1, faces), (s0, s1, sf)])


def nbody_scene(count=13200, size=0.4, motion=0.6, seed=3, big_fraction=0.01, big_scale=20.0) -> SceneStep:
    """C3: n-body-like box soup (bench.cpp:400-446 recipe, region
    1.2*cbrt(count)) plus 1% bodies at 20x size and two static container
    walls spanning the region, so a few sweep rows run to ~k."""
    region = 1.2 * count ** (1.0 / 3.0)
    rng = Rng(seed)
    v0, v1, f = _box_soup_arrays(count, region, size, motion, rng)
    nbig = max(1, int(round(count * big_fraction)))
    b0, b1, bf = _box_soup_arrays(nbig, region, size * big_scale, motion, rng)
    lo, hi = -1.0, region + 1.0
    wall = []
    for x in (lo, hi):
        w = np.array([[x, lo, lo], [x, hi, lo], [x, hi, hi], [x, lo, hi]])
        wall.append((w, w.copy(), np.array([[0, 1, 2], [0, 2, 3]], np.uint32)))
    floor = np.array([[lo, lo, lo], [hi, lo, lo], [hi, lo, hi], [lo, lo, hi]])
    wall.append((floor, floor.copy(), np.array([[0, 1, 2], [0, 2, 3]], np.uint32)))
    return _merge([(v0, v1, f), (b0, b1, bf)] + wall)


def _rotation(rng: Rng, n: int) -> np.ndarray:
    q = rng.doubles(4 * n).reshape(n, 4) * 2.0 - 1.0
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)], -1),
        np.stack([2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)], -1),
        np.stack([2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], -1),
    ], 1)


def degenerate_queries(n: int, seed: int = 2024, n_exhaust: int = 0) -> QueryBatch:
    """Near-degenerate families under a generic rotation: plane crossings
    (helpers.hpp:46-53), tangent double roots (test_oracle.cpp:63-66),
    parallel-above (test_narrowphase.cpp:113-115), coincident (58-60), and
    VF/EE slides at gaps 1e-2/1e-3/1e-4; the last ``n_exhaust`` are slides at
    gap 2e-6 that exhaust the 2^20 split budget."""
    rng = Rng(seed)
    rot = _rotation(rng, n)
    shift = rng.doubles(3 * n).reshape(n, 3)
    jig = rng.doubles(4 * n).reshape(n, 4)
    kind = np.zeros(n, np.uint8)
    base = np.zeros((n, 2, 4, 3))
    tri = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]])
    for i in range(n):
        fam = i % 8 if i < n - n_exhaust else 8 + (i % 2)
        a, b = 0.1 + 0.3 * jig[i, 0], 0.1 + 0.3 * jig[i, 1]
        if fam == 0:  # plane crossing
            base[i, 0, 0] = [a, b, 1.0]
            base[i, 1, 0] = [a, b, -1.0]
            base[i, :, 1:] = tri
        elif fam == 1:  # tangent double root
            base[i, 0] = [[0.25, 0.25, -1], [0, 0, 0], [1, 0, -1], [0, 1, -1]]
            base[i, 1] = [[1.25, 0.25, 1], [0, 0, 0], [1, 0, 1], [0, 1, 1]]
        elif fam == 2:  # parallel above
            base[i, 0, 0] = [a, b, 1.0]
            base[i, 1, 0] = [a + 0.4, b, 1.0]
            base[i, :, 1:] = tri
        elif fam == 3:  # coincident
            kind[i] = jig[i, 2] < 0.5
        elif fam in (4, 5, 6, 7) or fam in (8, 9):
            gap = {4: 1e-2, 5: 1e-3, 6: 1e-4, 7: 1e-3, 8: 2e-6, 9: 2e-6}[fam]
            if fam in (7, 9):  # EE: parallel edges sliding past at a gap
                kind[i] = 1
                base[i, 0] = [[0, 0, gap], [1, 0, gap], [0.2, -0.5, 0], [0.2, 0.5, 0]]
                base[i, 1] = [[0.5, 0, gap], [1.5, 0, gap], [0.2, -0.5, 0], [0.2, 0.5, 0]]
                base[i, 1, 0:2, 2] = gap
            else:  # VF slide across the face at a gap
                base[i, 0, 0] = [0.05, 0.05 + 0.3 * jig[i, 3], gap]
                base[i, 1, 0] = [0.6, 0.05 + 0.3 * jig[i, 3], gap]
                base[i, :, 1:] = tri
    pts = np.einsum("nij,nspj->nspi", rot, base) + shift[:, None, None, :]
    return QueryBatch(kind, np.ascontiguousarray(pts.reshape(n, 24)))


def mixed_queries(n: int, seed: int = 1003, every: int = 10000, n_exhaust: int = 16) -> QueryBatch:
    """C5: ``random_queries(n)`` with every ``every``-th query replaced by a
    rotated near-degenerate family member; ``n_exhaust`` of those are
    budget-exhausting slides at gap 2e-6."""
    qb = random_queries(n, seed)
    idx = np.arange(every - 1, n, every)
    if idx.size:
        deg = degenerate_queries(idx.size, seed=seed + 1, n_exhaust=min(n_exhaust, idx.size))
        qb.kind[idx] = deg.kind
        qb.points[idx] = deg.points
    return qb


CONFIGS = {
    "C1": "cloth-on-sphere 100x100 (+icosphere s4 r30), seed 1",
    "C2": "cloth-ball-like 224x224 pleated self-contact + ball, seed 2",
    "C3": "n-body-like box soup 13200 (+1% 20x bodies, 3 static walls), seed 3",
    "C4": "armadillo-rollers-like ~1M primitives = make_cloth_scene(410,410,.02,1,4)",
    "C5": "10M mixed VF/EE narrow-phase queries (Rng 1003) + rotated near-degenerates",
}


def config_scene(name: str, scale: float = 1.0) -> SceneStep:
    """Scenes for C1-C4.  ``scale`` < 1 shrinks the grid/body counts for
    quick parity runs (same recipe)."""
    if name == "C1":
        n = max(4, int(round(100 * math.sqrt(scale))))
        return cloth_on_sphere(n, n)
    if name == "C2":
        n = max(6, int(round(224 * math.sqrt(scale))))
        return cloth_ball(n)
    if name == "C3":
        return nbody_scene(max(8, int(round(13200 * scale))))
    if name == "C4":
        n = max(4, int(round(410 * math.sqrt(scale))))
        return make_cloth_scene(n, n, 0.02, 1.0, 4)
    raise KeyError(name)


def config_queries(n: int = 10_000_000) -> QueryBatch:
    return mixed_queries(n)
