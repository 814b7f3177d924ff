"""Exact ground truth for the narrow phase (oracle/exact_roots.py, a
restatement of the reference's GMP oracle, proj/src/oracle.cpp:285-691).

CPU: the oracle's own known answers (proj/tests/test_oracle.cpp).
GPU: conservativeness of the B200 narrow phase against the exact first-contact
times — no query whose exact first valid root lies in [0, 1] may report a ToI
after it (zero false negatives, the north star's narrow-phase bar), on random
queries and the rotated near-degenerate families of BASELINE config 5.
"""
import numpy as np
import pytest

from fixtures import plane_crossing_query
from oracle.exact_roots import exact_first_contact
from paper_2112_06300_b200 import ccdkit as ck, scenes


def _q(p0, p1):
    return np.array(p0 + p1, np.float64).reshape(24)


def test_plane_crossing_root_is_exactly_half():
    q = plane_crossing_query()
    status, lo, hi = exact_first_contact(0, q.points[0])
    assert status == "contact" and lo == hi == 0.5  # test_oracle.cpp:12-22


def test_parallel_pass_above_has_no_root():
    p0 = [[0.2, 0.2, 1.0], [0, 0, 0], [1, 0, 0], [0, 1, 0]]
    p1 = [[0.6, 0.2, 1.0], [0, 0, 0], [1, 0, 0], [0, 1, 0]]
    assert exact_first_contact(0, _q(p0, p1))[0] == "none"  # test_oracle.cpp:24-36


def test_tangential_double_root_collides_at_half():
    p0 = [[0.25, 0.25, -1], [0, 0, 0], [1, 0, -1], [0, 1, -1]]
    p1 = [[1.25, 0.25, 1], [0, 0, 0], [1, 0, 1], [0, 1, 1]]
    status, lo, hi = exact_first_contact(0, _q(p0, p1))
    assert status == "contact" and lo == hi == 0.5  # test_oracle.cpp:58-71


def test_irrational_root_is_bracketed():
    p0 = [[0.3, 0.2, 1.0], [0, 0, 0], [1, 0, 0], [0, 1, 0]]
    p1 = [[0.2, 0.3, -1.0], [0, 0.1, 0.2], [1.1, 0, -0.1], [0, 1, 0.1]]
    status, lo, hi = exact_first_contact(0, _q(p0, p1))
    assert status == "contact" and 0 <= lo <= hi <= 1  # test_oracle.cpp:38-56


def test_edge_edge_crossing():
    # two segments crossing at t = 0.5 at their midpoints
    p0 = [[0, 0, 1], [1, 0, 1], [0.5, -0.5, 0], [0.5, 0.5, 0]]
    p1 = [[0, 0, -1], [1, 0, -1], [0.5, -0.5, 0], [0.5, 0.5, 0]]
    status, lo, hi = exact_first_contact(1, _q(p0, p1))
    assert status == "contact" and lo == hi == 0.5


def test_reference_is_conservative_against_exact_roots(ref):
    """The parity target itself (the unmodified reference, oracle/_ref) never
    reports a ToI after the exact first contact (acceptance.cpp:165-198)."""
    qb = scenes.random_queries(300, seed=33)
    toi, _, _ = ref.narrow_phase(qb.kind, qb.points, ck.NarrowConfig().to_c())
    contacts = 0
    for i in range(len(qb)):
        status, lo, hi = exact_first_contact(int(qb.kind[i]), qb.points[i])
        if status == "contact":
            contacts += 1
            assert toi[i] <= float(hi), i
    assert contacts > 10


@pytest.mark.gpu
def test_zero_false_negatives_against_exact_roots(ctx):
    qb = scenes.random_queries(2500, seed=1003)
    deg = scenes.degenerate_queries(160, seed=2024)
    kind = np.concatenate([qb.kind, deg.kind])
    pts = np.concatenate([qb.points, deg.points])
    got = ck.narrow_phase(scenes.QueryBatch(kind, pts), ctx=ctx)
    contacts = violations = undecided = 0
    for i in range(len(kind)):
        status, lo, hi = exact_first_contact(int(kind[i]), pts[i])
        if status == "contact":
            contacts += 1
            # conservative: reported ToI never after the true first contact
            if not got.toi[i] <= float(hi):
                violations += 1
        elif status == "indeterminate":
            undecided += 1
    assert violations == 0
    assert contacts > 100            # the sample really exercises contacts
    assert undecided < len(kind) // 10
