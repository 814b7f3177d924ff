"""CPU suite: pin the C restatement (oracle/liborc.so) to the reference.

The reference itself (oracle/_ref/libccdref.so, compiled from the unmodified
sources) is the ground truth; the restatement must agree bit for bit, and
both must reproduce the known answers of the reference's own tests
(BASELINE.md §4).
"""
import numpy as np
import pytest

from paper_2112_06300_b200 import abi, scenes

from fixtures import (plane_crossing_query, plane_crossing_scene, random_boxes, random_subboxes,
                      random_triangle_soup, special_doubles)


def b64(x):
    return np.ascontiguousarray(x).view(np.uint64)


def test_known_answers_restatement(orc):
    d, u = orc.round_reduced(np.array([0.1, 0.0, 1.0, -2.5]))
    assert d.view(np.uint32)[0] == 0x3DCCCCCC and u.view(np.uint32)[0] == 0x3DCCCCCD
    assert d[1:].tolist() == [0.0, 1.0, -2.5] and u[1:].tolist() == [0.0, 1.0, -2.5]
    q = plane_crossing_query()
    r = orc.inclusion_box(0, q.points[0], np.array([0, 1, 0, 1, 0, 1.0]))
    assert r[4] == -float.fromhex("0x1.0000000000008p+0") and r[5] == float.fromhex("0x1.0000000000004p+0")
    toi, flags, st = orc.narrow_phase(q.kind, q.points, abi.narrow_cfg())
    assert toi[0] == 0.5 - 2.0 ** -21 and st.total_splits == 449 and st.peak_queue == 16
    toi, flags, st = orc.narrow_phase(q.kind, q.points, abi.narrow_cfg(min_separation=0.25))
    assert toi[0] == 0.37451171875
    toi, flags, st = orc.narrow_phase(q.kind, q.points, abi.narrow_cfg(max_splits=4))
    assert toi[0] == 0.25 and flags[0] == abi.FLAG_TOLERANCE_HIT
    k3 = np.zeros(3, np.uint8)
    p3 = np.repeat(q.points, 3, axis=0)
    _, _, st = orc.narrow_phase(k3, p3, abi.narrow_cfg(), capacity=2)
    assert st.overflow
    # parallel-above query is pruned at the root (test_narrowphase.cpp:110-124)
    pa = q.points.copy()
    pa[0, 0:3] = [0.2, 0.2, 1.0]
    pa[0, 12:15] = [0.6, 0.2, 1.0]
    toi, _, st = orc.narrow_phase(q.kind, pa, abi.narrow_cfg())
    assert np.isinf(toi[0]) and st.total_splits == 0


def test_generators_match_reference(ref):
    for args in [(30, 30, 0.02, 1.0, 1), (7, 5, 0.1, 0.5, 9)]:
        a, b = ref.make_scene("cloth", *args), scenes.make_cloth_scene(*args)
        for x, y in [(a.vertices_t0, b.vertices_t0), (a.vertices_t1, b.vertices_t1),
                     (a.edges, b.edges), (a.faces, b.faces)]:
            np.testing.assert_array_equal(x.view(np.uint8), y.view(np.uint8))
    for args in [(30, 4.0, 0.4, 1.0, 5), (64, 8.0, 0.45, 0.9, 42)]:
        a, b = ref.make_scene("soup", *args), scenes.make_box_soup(*args)
        for x, y in [(a.vertices_t0, b.vertices_t0), (a.vertices_t1, b.vertices_t1),
                     (a.edges, b.edges), (a.faces, b.faces)]:
            np.testing.assert_array_equal(x.view(np.uint8), y.view(np.uint8))


def test_rounding_restatement(ref, orc):
    x = special_doubles(3, 3000)
    a, b = ref.round_reduced(x), orc.round_reduced(x)
    np.testing.assert_array_equal(a[0].view(np.uint32), b[0].view(np.uint32))
    np.testing.assert_array_equal(a[1].view(np.uint32), b[1].view(np.uint32))


@pytest.mark.parametrize("inflation", [0.0, 0.01])
def test_boxes_restatement(ref, orc, inflation):
    for s in [scenes.make_cloth_scene(25, 20, 0.02, 1.0, 2), random_triangle_soup(3, 500)]:
        for x, y in zip(ref.build_boxes(s, inflation), orc.build_boxes(s, inflation)):
            np.testing.assert_array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))


def test_broad_restatement(ref, orc):
    for trial in range(8):
        b, s = random_boxes(300 + trial, 50 + 70 * trial)
        for m in (abi.BROAD_STQ, abi.BROAD_SAP, abi.BROAD_BF):
            for rng in [(0, abi.UINT64_MAX), (10, len(b) // 2)]:
                pa, ra, qa = ref.broad(m, b.as_tuple(), s, *rng)
                pb, rb, qb = orc.broad(m, b.as_tuple(), s, *rng)
                np.testing.assert_array_equal(pa, pb)
                if m == abi.BROAD_STQ:
                    np.testing.assert_array_equal(ra, rb)
                    assert qa == qb
    s = scenes.make_cloth_scene(30, 30, 0.02, 1.0, 1)
    boxes = ref.build_boxes(s, 0.01)
    assert ref.choose_axis(boxes[0], boxes[1]) == orc.choose_axis(boxes[0], boxes[1])
    pa, _, _ = ref.broad(abi.BROAD_STQ, boxes, s)
    pb, _, _ = orc.broad(abi.BROAD_SAP, boxes, s)
    np.testing.assert_array_equal(pa, pb)
    ka, pta, sa, na = ref.classify(pa, s)
    kb, ptb, sb, nb = orc.classify(pa, s)
    assert na == nb
    np.testing.assert_array_equal(ka, kb)
    np.testing.assert_array_equal(b64(pta), b64(ptb))
    np.testing.assert_array_equal(sa, sb)


def test_inclusion_and_process_restatement(ref, orc):
    qb = scenes.random_queries(300, seed=31)
    boxes, depth = random_subboxes(32, 300)
    cfg = abi.narrow_cfg(delta=0.05)
    for i in range(300):
        a = ref.inclusion_box(qb.kind[i], qb.points[i], boxes[i])
        b = orc.inclusion_box(qb.kind[i], qb.points[i], boxes[i])
        np.testing.assert_array_equal(b64(a), b64(b))
        ra = ref.process_interval(qb.kind[i], qb.points[i], boxes[i], depth[i], np.inf, -1.0, cfg)
        rb = orc.process_interval(qb.kind[i], qb.points[i], boxes[i], depth[i], np.inf, -1.0, cfg)
        assert ra[0] == rb[0] and ra[2] == rb[2]
        np.testing.assert_array_equal(b64(np.array([ra[1]])), b64(np.array([rb[1]])))
        np.testing.assert_array_equal(b64(ra[3]), b64(rb[3]))
        np.testing.assert_array_equal(ra[4], rb[4])


@pytest.mark.parametrize("cfg", [abi.narrow_cfg(), abi.narrow_cfg(max_splits=37),
                                 abi.narrow_cfg(max_splits=3, no_zero_toi=1),
                                 abi.narrow_cfg(min_separation=0.01, t_max=0.6)])
def test_narrow_restatement(ref, orc, cfg):
    qb = scenes.random_queries(600, seed=33)
    ta, fa, sa = ref.narrow_phase(qb.kind, qb.points, cfg)
    tb, fb, sb = orc.narrow_phase(qb.kind, qb.points, cfg)
    np.testing.assert_array_equal(b64(ta), b64(tb))
    np.testing.assert_array_equal(fa, fb)
    assert (sa.peak_queue, sa.total_splits, sa.overflow) == (sb.peak_queue, sb.total_splits, sb.overflow)


def test_ccd_restatement(ref, orc):
    for s in [scenes.make_cloth_scene(20, 20, 0.02, 1.0, 1), scenes.make_box_soup(25, 4.0, 0.4, 1.0, 6),
              plane_crossing_scene()]:
        cfg = abi.pipeline_cfg(inflation=0.01)
        ra, pa = ref.ccd(s, cfg)
        rb, pb = orc.ccd(s, cfg)
        np.testing.assert_array_equal(pa, pb)
        assert ra.toi == rb.toi and ra.candidate_count == rb.candidate_count
        assert ra.query_count == rb.query_count and ra.tolerance_hit == rb.tolerance_hit


def test_ref_run_batched_adapter(ref, orc):
    """The adapter's run_batched (the GPU tests' reference for ccdk_run_batched)
    on the scene's own boxes reproduces ccd (pipeline.cpp:218-232 is exactly
    build_boxes + run_batched); with a small budget the union is the same set
    and the trace counts the batches that ran."""
    s = scenes.make_cloth_scene(20, 20, 0.02, 1.0, 1)
    cfg = abi.pipeline_cfg(inflation=0.01)
    boxes = orc.build_boxes(s, 0.01)
    ra, pa = ref.ccd(s, cfg)
    rb, pb, bb, nb = ref.run_batched(s, boxes, cfg)
    np.testing.assert_array_equal(pa, pb)
    assert (ra.toi, ra.candidate_count, ra.query_count, ra.batch_count) == \
        (rb.toi, rb.candidate_count, rb.query_count, rb.batch_count)
    assert (bb, nb) == (1, 1) and rb.tracked_peak_bytes == ra.tracked_peak_bytes
    small = abi.pipeline_cfg(inflation=0.01, memory_budget=1 << 19)
    rc, pc, bb, nb = ref.run_batched(s, boxes, small)
    np.testing.assert_array_equal(pc, pa)
    assert rc.toi == ra.toi and bb > 1 and nb >= bb and rc.batch_count == nb
