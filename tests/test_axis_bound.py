"""choose_axis near-tie certification (CPU, no GPU needed).

K2 sums box centres and squared deviations in a fixed-shape tree
(ccdk_broad.cu k_axis_sum / k_axis_var / k_axis_pick); the reference sums
serially (proj/src/broadphase.cpp:45-67).  k_axis_pick certifies the tree's
argmax with an error bound and flags near ties for the serial recomputation
(k_axis_serial).  This file emulates the tree reduction bit for bit in numpy
and checks, against the reference compiled here (oracle/_ref), that every
input on which the two orders disagree is flagged, and that the BASELINE-
style jittered scenes are not (so the step never pays for the serial pass).
"""
import numpy as np
import pytest

from paper_2112_06300_b200 import scenes

R_BLOCKS = 256
R_THREADS = 256
U = 2.0 ** -53


def _block_tree(v):
    """block_sum3's shared-memory tree over 256 thread values."""
    v = v.copy()
    w = R_THREADS // 2
    while w > 0:
        v[:w] = v[:w] + v[w:2 * w]
        w //= 2
    return v[0]


def _grid_partials(vals):
    """Per-thread grid-stride serial sums, then each block's tree."""
    k = vals.shape[0]
    stride = R_BLOCKS * R_THREADS
    pad = (-k) % stride
    x = np.concatenate([vals, np.zeros(pad)]).reshape(-1, stride)
    acc = np.zeros(stride)
    for row in x:  # serial per thread, in grid-stride order
        acc = acc + row
    acc = acc.reshape(R_BLOCKS, R_THREADS)
    return np.array([_block_tree(acc[b]) for b in range(R_BLOCKS)])


def _final(part):
    # k_axis_pick / mean_from_partials: one partial per thread (256 == blocks), then the tree
    return _block_tree(part)


def gpu_axis(mn, mx):
    """Bit-exact emulation of k_axis_sum/var/pick: (axis, near_tie)."""
    k = mn.shape[0]
    c = (mn.astype(np.float64) + mx.astype(np.float64)) / 2.0
    var, asum = [], []
    for a in range(3):
        s = _final(_grid_partials(c[:, a]))
        m = s / float(k)
        d = c[:, a] - m
        var.append(_final(_grid_partials(d * d)))
        asum.append(_final(_grid_partials(np.abs(c[:, a]))))
    best = 0
    for a in (1, 2):
        if var[a] > var[best]:
            best = a

    def gamma(m):
        return m * U / (1.0 - m * U)

    n = float(k)
    g = gamma(n + 3.0)
    R = []
    for a in range(3):
        dm = gamma(n + 2.0) * asum[a] * (1.0 + 4.0 * g) / n
        R.append(4.0 * g * var[a] + 4.0 * n * dm * dm + 2.0 ** -1000)
    tie = any(a != best and var[best] - R[best] <= var[a] + R[a] for a in range(3))
    return best, tie


def _boxes(ref, s):
    mn, mx, _, _ = ref.build_boxes(s, 0.01)
    return mn, mx


UNJITTERED = [(n, off) for n in (30, 41, 64, 100) for off in (0.0, 1.0)]


@pytest.mark.parametrize("n,drop", UNJITTERED)
def test_unjittered_cloth_divergence_is_flagged(ref, n, drop):
    s = scenes.make_cloth_scene(n, n, 0.0, drop, 1)
    mn, mx = _boxes(ref, s)
    serial = ref.choose_axis(mn, mx)
    tree, tie = gpu_axis(mn, mx)
    if tree != serial:
        assert tie, (n, drop, tree, serial)


def test_some_unjittered_cloth_really_diverges(ref):
    # the failure the certification exists for (30x30 cloth, axis 2 vs 0)
    s = scenes.make_cloth_scene(30, 30, 0.0, 1.0, 1)
    mn, mx = _boxes(ref, s)
    tree, tie = gpu_axis(mn, mx)
    assert ref.choose_axis(mn, mx) == 2 and tree == 0 and tie


@pytest.mark.parametrize("n,seed", [(60, 1), (100, 4), (150, 2)])
def test_jittered_cloth_not_flagged(ref, n, seed):
    s = scenes.make_cloth_scene(n, n, 0.02, 1.0, seed)
    mn, mx = _boxes(ref, s)
    tree, tie = gpu_axis(mn, mx)
    assert not tie
    assert tree == ref.choose_axis(mn, mx)


def test_exact_equal_variances_flagged(ref):
    # two axes with bit-identical centre columns: a true tie, serial picks the lower
    rng = np.random.default_rng(5)
    c = rng.random((5000, 1)).astype(np.float32)
    mn = np.hstack([c, c, c * 0.5]).astype(np.float32)
    mx = mn + np.float32(0.01)
    tree, tie = gpu_axis(mn, mx)
    assert tie and ref.choose_axis(mn, mx) == 0
