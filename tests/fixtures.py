"""Input fixtures restating the reference tests' generators (seeded splitmix64)."""
from __future__ import annotations

import numpy as np

from paper_2112_06300_b200.ccdkit import Boxes
from paper_2112_06300_b200.scenes import QueryBatch, Rng, SceneStep


def random_boxes(seed: int, n: int, stretch=(1.0, 1.0, 1.0)):
    """test_broadphase.cpp:22-56 / acceptance.cpp:41-75: isolated primitives
    (n/2 vertices, the rest single-triangle faces on their own vertices) whose
    boxes are placed freely: lo = U[0,10)*s, size = U[0,2)*s per axis."""
    rng = Rng(seed)
    d = rng.doubles(6 * n).reshape(n, 3, 2)
    s = np.asarray(stretch, np.float64)
    lo = (0.0 + 10.0 * d[:, :, 0]) * s
    size = (0.0 + 2.0 * d[:, :, 1]) * s
    mn = lo.astype(np.float32)
    mx = (lo + size).astype(np.float32)
    n_verts = n // 2
    verts, faces, kind, index = [], [], [], []
    for i in range(n):
        if i < n_verts:
            kind.append(0)
            index.append(len(verts))
            verts.append(lo[i])
        else:
            base = len(verts)
            verts += [lo[i]] * 3
            kind.append(2)
            index.append(len(faces))
            faces.append((base, base + 1, base + 2))
    v = np.array(verts, np.float64).reshape(-1, 3)
    f = np.array(faces, np.uint32).reshape(-1, 3)
    scene = SceneStep(v, v.copy(), np.zeros((0, 2), np.uint32), f)
    return Boxes(mn, mx, np.array(kind, np.uint8), np.array(index, np.uint32)), scene


def random_triangle_soup(seed: int, triangles: int) -> SceneStep:
    """test_geometry.cpp:87-105: coordinates spanning 1e-3..1e3 scales."""
    rng = Rng(seed)
    d = rng.doubles(triangles * 3 * 3 * 3).reshape(triangles, 3, 3, 3)
    p0 = (-10.0 + 20.0 * d[..., 0]) * np.power(10.0, -3.0 + 6.0 * d[..., 1])
    p1 = p0 + (-1.0 + 2.0 * d[..., 2])
    v0 = p0.reshape(-1, 3)
    v1 = p1.reshape(-1, 3)
    base = 3 * np.arange(triangles, dtype=np.uint32)
    f = np.stack([base, base + 1, base + 2], 1)
    e = np.concatenate([np.stack([base, base + 1], 1), np.stack([base + 1, base + 2], 1),
                        np.stack([base, base + 2], 1)])
    return SceneStep(v0, v1, e, f)


def random_subboxes(seed: int, n: int):
    """test_narrowphase.cpp:37-54: dyadic sub-boxes of [0,1]^3, depth < 6."""
    rng = Rng(seed)
    boxes = np.zeros((n, 6))
    depth = np.zeros((n, 3), np.uint16)
    z = rng.u64(n * 3 * 7).reshape(n, 3, 7)
    for i in range(n):
        for d in range(3):
            k = int(z[i, d, 0] % np.uint64(6))
            lo, hi = 0.0, 1.0
            for s in range(k):
                mid = lo + 0.5 * (hi - lo)
                if int(z[i, d, 1 + s] % np.uint64(2)):
                    lo = mid
                else:
                    hi = mid
            boxes[i, 2 * d], boxes[i, 2 * d + 1] = lo, hi
            depth[i, d] = k
    return boxes, depth


def plane_crossing_scene() -> SceneStep:
    """tests/helpers.hpp:36-44."""
    v0 = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0.25, 0.25, 1]], np.float64)
    v1 = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0.25, 0.25, -1]], np.float64)
    return SceneStep(v0, v1, np.array([[0, 1], [0, 2], [1, 2]], np.uint32),
                     np.array([[0, 1, 2]], np.uint32))


def plane_crossing_query() -> QueryBatch:
    """tests/helpers.hpp:46-53."""
    p0 = [[0.25, 0.25, 1], [0, 0, 0], [1, 0, 0], [0, 1, 0]]
    p1 = [[0.25, 0.25, -1], [0, 0, 0], [1, 0, 0], [0, 1, 0]]
    return QueryBatch(np.zeros(1, np.uint8), np.array([p0 + p1], np.float64).reshape(1, 24))


def concat(*qbs: QueryBatch) -> QueryBatch:
    return QueryBatch(np.concatenate([q.kind for q in qbs]), np.concatenate([q.points for q in qbs]))


def special_doubles(seed: int, n: int) -> np.ndarray:
    """Random bit patterns, magnitudes 2^+-170 and float-boundary specials."""
    rng = Rng(seed)
    z = rng.u64(n)
    raw = z.view(np.float64)
    raw = raw[np.isfinite(raw)]
    d = rng.doubles(2 * n).reshape(n, 2)
    scaled = (d[:, 0] * 2 - 1) * np.exp2(np.floor(-170 + 340 * d[:, 1]))
    f32 = np.float32
    specials = np.array([0.0, -0.0, 1.0, -2.5, 0.1, -0.1, 3.4028234663852886e38, 3.5e38, -3.5e38,
                         1e300, -1e300, 1e-40, -1e-40, 1e-46, -1e-46, 5e-324, -5e-324,
                         float(np.nextafter(f32(1), f32(2))), 2.0 ** -149, 2.0 ** -150, 2.0 ** -126],
                        np.float64)
    return np.concatenate([specials, raw, scaled])
