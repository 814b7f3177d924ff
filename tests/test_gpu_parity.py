"""GPU parity: the sm_100a path (through the C ABI) against the CPU checkers.

The checkers are the reference itself (oracle/_ref, bit-exact target) and our
C restatement (oracle/liborc.so).  Bars (SURVEY §8 / BASELINE.md §4):
  * boxes, rounding, candidate sets, round sizes: bit-exact;
  * inclusion boxes, process_interval, per-query ToI and flags, total_splits,
    peak_queue: bit-exact (stronger than the north star's "ToI within delta,
    zero false negatives", which bit-exactness implies).
"""
import numpy as np
import pytest

from paper_2112_06300_b200 import abi, ccdkit as ck, scenes
from paper_2112_06300_b200.ccdkit import NarrowConfig, PipelineConfig, SweepRange

from fixtures import (concat, plane_crossing_query, plane_crossing_scene, random_boxes,
                      random_subboxes, random_triangle_soup, special_doubles)

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def assert_bits(a, b):
    assert a.shape == b.shape
    np.testing.assert_array_equal(bits(a), bits(b))


# ------------------------------------------------------------------ geometry

def test_rounding_matches_reference(ctx, orc):
    x = special_doubles(7, 20000)
    dn, up = ck.round_reduced(x, ctx)
    edn, eup = orc.round_reduced(x)
    assert_bits(dn, edn)
    assert_bits(up, eup)
    assert ck.round_down_reduced(0.1, ctx).view(np.uint32) == 0x3DCCCCCC
    assert ck.round_up_reduced(0.1, ctx).view(np.uint32) == 0x3DCCCCCD


def test_rounding_rejects_non_finite(ctx):
    with pytest.raises(ck.InvalidInput):
        ck.round_reduced(np.array([1.0, np.nan]), ctx)
    with pytest.raises(ck.InvalidInput):
        ck.round_reduced(np.array([np.inf]), ctx)


@pytest.mark.parametrize("inflation", [0.0, 0.01, 0.5])
def test_build_boxes_bit_exact(ctx, ref, inflation):
    for s in [scenes.make_cloth_scene(20, 17, 0.02, 1.0, 3), scenes.make_box_soup(50, 6.0, 0.4, 0.9, 11),
              random_triangle_soup(5, 3000)]:
        got = ck.build_boxes(s, inflation, ctx=ctx)
        exp = ref.build_boxes(s, inflation)
        for g, e in zip(got.as_tuple(), exp):
            np.testing.assert_array_equal(np.asarray(g).view(np.uint8), np.asarray(e).view(np.uint8))


def test_build_boxes_known_answers(ctx):
    s = scenes.SceneStep([[0, 0, 0]], [[0, 0, 0]], np.zeros((0, 2)), np.zeros((0, 3)))
    b = ck.build_boxes(s, ctx=ctx)
    assert b.min_corner.tolist() == [[0, 0, 0]] and b.max_corner.tolist() == [[0, 0, 0]]
    s = scenes.SceneStep([[0, 0, 0], [1, 0, 0]], [[0, 0, 1], [1, 0, 1]], [[0, 1]], np.zeros((0, 3)))
    b = ck.build_boxes(s, ctx=ctx)
    assert len(b) == 3 and b.owner_kind[2] == ck.KIND_EDGE and b.owner_index[2] == 0
    assert b.min_corner[2].tolist() == [0, 0, 0] and b.max_corner[2].tolist() == [1, 0, 1]
    b = ck.build_boxes(scenes.SceneStep([[1, 2, 3]], [[1, 2, 3]], np.zeros((0, 2)), np.zeros((0, 3))), 0.1, ctx=ctx)
    assert (b.max_corner[0].astype(np.float64) - b.min_corner[0] >= 2e-12).all()


def test_scene_validation_errors(ctx):
    good = plane_crossing_scene()
    bad = scenes.SceneStep(good.vertices_t0, good.vertices_t1, [[0, 7]], good.faces)
    with pytest.raises(ck.InvalidInput):
        ck.build_boxes(bad, ctx=ctx)
    bad = scenes.SceneStep(good.vertices_t0, good.vertices_t1, [[1, 1]], good.faces)
    with pytest.raises(ck.InvalidInput):
        ck.build_boxes(bad, ctx=ctx)
    v = good.vertices_t0.copy()
    v[0, 0] = np.nan
    with pytest.raises(ck.InvalidInput):
        ck.ccd(scenes.SceneStep(v, good.vertices_t1, good.edges, good.faces), ctx=ctx)
    with pytest.raises(ck.ConfigError):
        ck.ccd(good, PipelineConfig(narrow=NarrowConfig(delta=0.0)), ctx=ctx)


# -------------------------------------------------------------- broad phase

def test_choose_axis(ctx, ref):
    b, _ = random_boxes(21, 1000, (1, 1, 100))
    assert ck.choose_axis(b, ctx) == 2 == ref.choose_axis(b.min_corner, b.max_corner)
    with pytest.raises(ck.InvalidInput):
        ck.choose_axis(ck.Boxes(np.zeros((0, 3), np.float32), np.zeros((0, 3), np.float32),
                                np.zeros(0, np.uint8), np.zeros(0, np.uint32)), ctx)
    for seed in range(5):
        b, _ = random_boxes(100 + seed, 3000, (1.0, 1.3, 0.7))
        assert ck.choose_axis(b, ctx) == ref.choose_axis(b.min_corner, b.max_corner)


def test_stq_trivial(ctx):
    b, s = random_boxes(22, 2)
    b.min_corner[:] = [[0, 0, 0], [1, 1, 5]]
    b.max_corner[:] = [[2, 2, 1], [3, 3, 6]]
    assert ck.stq(b, s, ctx=ctx).shape == (0, 2)
    b.min_corner[1] = b.min_corner[0]
    b.max_corner[1] = b.max_corner[0]
    b.owner_kind[:] = [0, 2]
    b.owner_index[:] = [0, 0]
    pairs = ck.stq(b, s, ctx=ctx)
    assert pairs.tolist() == [[0, 2 << 32]]


@pytest.mark.parametrize("method", [abi.BROAD_STQ, abi.BROAD_SAP, abi.BROAD_BF])
def test_broad_phase_random_sets_bit_exact(ctx, ref, method):
    rng = scenes.Rng(25)
    for trial in range(40):
        n = 1 + int(rng.u64(1)[0] % np.uint64(600))
        b, s = random_boxes(1000 + trial, n)
        got = ck._broad(method, b, s, None, None, ctx)
        exp, _, _ = ref.broad(method, b.as_tuple(), s)
        np.testing.assert_array_equal(got, exp)


def test_stq_stats_and_ranges(ctx, ref):
    for trial in range(6):
        b, s = random_boxes(2000 + trial, 300 + 150 * trial)
        st = ck.StqStats()
        got = ck.stq(b, s, stats=st, ctx=ctx)
        exp, rounds, mq = ref.broad(abi.BROAD_STQ, b.as_tuple(), s)
        np.testing.assert_array_equal(got, exp)
        assert st.round_sizes == rounds.tolist() and st.max_queue == mq
        k = len(b)
        for lo, hi in [(0, k // 3), (k // 3, k), (5, 17), (k - 1, k + 5)]:
            st = ck.StqStats()
            got = ck.stq(b, s, stats=st, range=SweepRange(lo, hi), ctx=ctx)
            exp, rounds, mq = ref.broad(abi.BROAD_STQ, b.as_tuple(), s, lo, hi)
            np.testing.assert_array_equal(got, exp)
            assert st.round_sizes == rounds.tolist()
            got = ck.bf(b, s, range=SweepRange(lo, hi), ctx=ctx)
            exp, _, _ = ref.broad(abi.BROAD_BF, b.as_tuple(), s, lo, hi)
            np.testing.assert_array_equal(got, exp)


def test_broad_phase_on_scenes(ctx, ref):
    for s in [scenes.make_cloth_scene(40, 40, 0.02, 1.0, 1), scenes.make_box_soup(300, 8.0, 0.45, 0.9, 42),
              scenes.config_scene("C3", 0.01)]:
        b = ck.build_boxes(s, 0.01, ctx=ctx)
        st = ck.StqStats()
        got = ck.stq(b, s, stats=st, ctx=ctx)
        exp, rounds, mq = ref.broad(abi.BROAD_STQ, b.as_tuple(), s)
        np.testing.assert_array_equal(got, exp)
        assert st.round_sizes == rounds.tolist()


def test_classify_matches_reference(ctx, ref):
    s = scenes.make_box_soup(60, 5.0, 0.4, 1.0, 9)
    b = ck.build_boxes(s, 0.01, ctx=ctx)
    pairs = ck.stq(b, s, ctx=ctx)
    # add pairs the filter must drop: shared vertex, wrong kinds, reversed
    extra = np.array([[ck.pack_id(1, 0), ck.pack_id(1, 1)], [ck.pack_id(0, 0), ck.pack_id(0, 5)],
                      [ck.pack_id(2, 3), ck.pack_id(0, 0)], [ck.pack_id(0, 0), ck.pack_id(2, 0)]],
                     np.uint64)
    allp = np.concatenate([pairs, extra, pairs[::7]])
    got = ck.classify(allp, s, ctx=ctx)
    ek, ep, es, envf = ref.classify(allp, s)
    assert got.n_vf == envf
    np.testing.assert_array_equal(got.queries.kind, ek)
    assert_bits(got.queries.points, ep)
    np.testing.assert_array_equal(got.sources, es)
    bad = np.array([[ck.pack_id(0, 0), ck.pack_id(2, 99999)]], np.uint64)
    with pytest.raises(ck.InvalidInput):
        ck.classify(bad, s, ctx=ctx)


# -------------------------------------------------------------- narrow phase

def test_inclusion_box_bits(ctx, ref):
    q = plane_crossing_query()
    r = ck.inclusion_box(0, q.points[0], ctx=ctx)
    assert r[4] == -float.fromhex("0x1.0000000000008p+0") and r[5] == float.fromhex("0x1.0000000000004p+0")
    assert r[0] == -float.fromhex("0x1.8000000000008p-1") and r[1] == float.fromhex("0x1.0000000000004p-2")
    qb = scenes.random_queries(500, seed=31)
    boxes, _ = random_subboxes(31, 500)
    got = ck.inclusion_boxes(qb.kind, qb.points, boxes, ctx)
    exp = np.stack([ref.inclusion_box(qb.kind[i], qb.points[i], boxes[i]) for i in range(500)])
    assert_bits(got, exp)


def test_inclusion_box_extreme_magnitudes(ctx, ref):
    """Queries beyond 2^1000 take the bit-increment (Exact) widening path."""
    qb = scenes.random_queries(64, seed=77)
    pts = qb.points * np.where(np.arange(64)[:, None] % 2 == 0, 1e307, 1e-300)
    boxes, _ = random_subboxes(78, 64)
    got = ck.inclusion_boxes(qb.kind, pts, boxes, ctx)
    exp = np.stack([ref.inclusion_box(qb.kind[i], pts[i], boxes[i]) for i in range(64)])
    assert_bits(got, exp)


def test_process_interval_matches_reference(ctx, ref):
    n = 400
    qb = concat(scenes.random_queries(n - 1, seed=41), plane_crossing_query())
    boxes, depth = random_subboxes(42, n)
    rng = scenes.Rng(43)
    t_star = np.where(rng.doubles(n) < 0.3, rng.doubles(n), np.inf)
    for cfg in [NarrowConfig(), NarrowConfig(delta=0.3, min_separation=0.01, no_zero_toi=True),
                NarrowConfig(t_max=0.4)]:
        a, ct, zd, ch, cd = ck.process_intervals(qb.kind, qb.points, boxes, depth, t_star, cfg, ctx=ctx)
        for i in range(n):
            ea, ect, ezd, ech, ecd = ref.process_interval(qb.kind[i], qb.points[i], boxes[i], depth[i],
                                                          t_star[i], -1.0, cfg.to_c())
            assert a[i] == ea and zd[i] == ezd, i
            assert bits(np.array([ct[i]]))[0] == bits(np.array([ect]))[0]
            assert_bits(ch[i], ech)
            np.testing.assert_array_equal(cd[i], ecd)


def test_plane_crossing_known_answers(ctx):
    q = plane_crossing_query()
    out = ck.narrow_phase(q, ctx=ctx)
    assert out.toi[0] == 0.5 - 2.0 ** -21 and out.total_splits == 449 and out.peak_queue == 16
    out = ck.narrow_phase(q, NarrowConfig(min_separation=0.25), ctx=ctx)
    assert out.global_toi == 0.37451171875
    out = ck.narrow_phase(q, NarrowConfig(max_splits=4), ctx=ctx)
    assert out.toi[0] == 0.25 and out.flags[0] & abi.FLAG_TOLERANCE_HIT
    out = ck.narrow_phase(concat(q, q, q), queue_capacity=2, ctx=ctx)
    assert out.overflow and np.isinf(out.global_toi)
    empty = ck.narrow_phase(scenes.QueryBatch(np.zeros(0, np.uint8), np.zeros((0, 24))), ctx=ctx)
    assert np.isinf(empty.global_toi) and empty.toi.size == 0


def _narrow_equal(got, toi, flags, st):
    assert_bits(got.toi, toi)
    np.testing.assert_array_equal(got.flags, flags)
    assert got.overflow == bool(st.overflow)
    if not got.overflow:
        assert got.total_splits == st.total_splits
        assert got.peak_queue == st.peak_queue
        assert bits(np.array([got.global_toi]))[0] == bits(np.array([st.global_toi]))[0]


@pytest.mark.parametrize("max_splits", [1 << 20, 37, 8, 1])
def test_narrow_phase_random_bit_exact(ctx, ref, max_splits):
    qb = scenes.random_queries(3000, seed=1003)
    cfg = NarrowConfig(max_splits=max_splits)
    got = ck.narrow_phase(qb, cfg, ctx=ctx)
    _narrow_equal(got, *ref.narrow_phase(qb.kind, qb.points, cfg.to_c()))


def test_narrow_phase_separations_and_no_zero(ctx, ref):
    qb = scenes.random_queries(1500, seed=34)
    seps = np.abs(scenes.Rng(35).doubles(1500)) * 0.05
    for cfg, sp in [(NarrowConfig(min_separation=0.02), None), (NarrowConfig(), seps),
                    (NarrowConfig(no_zero_toi=True), None), (NarrowConfig(no_zero_toi=True, max_splits=50), seps),
                    (NarrowConfig(t_max=0.3, delta=1e-4), None)]:
        got = ck.narrow_phase(qb, cfg, per_query_min_sep=sp, ctx=ctx)
        _narrow_equal(got, *ref.narrow_phase(qb.kind, qb.points, cfg.to_c(), seps=sp))


def test_narrow_phase_degenerate_families(ctx, ref):
    qb = scenes.degenerate_queries(64, seed=5)
    cfg = NarrowConfig(max_splits=20000)
    got = ck.narrow_phase(qb, cfg, ctx=ctx)
    _narrow_equal(got, *ref.narrow_phase(qb.kind, qb.points, cfg.to_c()))


def test_narrow_phase_capacity_semantics(ctx, ref):
    qb = scenes.random_queries(200, seed=8)
    for cap in [150, 300, 5000]:
        got = ck.narrow_phase(qb, NarrowConfig(), queue_capacity=cap, ctx=ctx)
        toi, flags, st = ref.narrow_phase(qb.kind, qb.points, NarrowConfig().to_c(), capacity=cap)
        assert got.overflow == bool(st.overflow), cap
        if not st.overflow:
            _narrow_equal(got, toi, flags, st)


def test_narrow_phase_physical_halving(ctx, ref):
    """A tiny device interval buffer forces the batch-halving path; per-query
    results stay bit-exact (each query's result depends only on itself)."""
    qb = scenes.random_queries(400, seed=9)
    ctx.set_interval_capacity(512)
    try:
        got = ck.narrow_phase(qb, ctx=ctx)
    finally:
        ctx.set_interval_capacity(0)
    toi, flags, st = ref.narrow_phase(qb.kind, qb.points, NarrowConfig().to_c())
    assert_bits(got.toi, toi)
    np.testing.assert_array_equal(got.flags, flags)
    assert got.total_splits == st.total_splits


# ------------------------------------------------------------------ pipeline

@pytest.mark.parametrize("name", ["cloth30", "soup", "C1", "C2", "C3", "C4"])
def test_ccd_matches_reference(ctx, ref, name):
    s = {"cloth30": lambda: scenes.make_cloth_scene(30, 30, 0.02, 1.0, 1),
         "soup": lambda: scenes.make_box_soup(40, 5.0, 0.4, 1.0, 1005),
         "C1": lambda: scenes.config_scene("C1", 0.05),
         "C2": lambda: scenes.config_scene("C2", 0.01),
         "C3": lambda: scenes.config_scene("C3", 0.004),
         "C4": lambda: scenes.config_scene("C4", 0.004)}[name]()
    cfg = PipelineConfig(inflation=0.01)
    got = ck.ccd(s, cfg, ctx=ctx)
    exp, pairs = ref.ccd(s, cfg.to_c())
    np.testing.assert_array_equal(got.candidates, pairs)
    assert got.candidate_count == exp.candidate_count and got.query_count == exp.query_count
    assert bits(np.array([got.toi.toi]))[0] == bits(np.array([exp.toi]))[0]
    assert got.toi.tolerance_hit == bool(exp.tolerance_hit)
    assert got.tracked_peak_bytes == exp.tracked_peak_bytes
    assert set(got.per_stage_times) == {"CB", "BP", "SO/CD", "NP"}


def test_ccd_trivial_scenes(ctx):
    s = scenes.SceneStep([[0, 0, 0], [1, 0, 0], [0, 1, 0], [50, 0, 0], [51, 0, 0], [50, 1, 0]],
                         [[0, 0, 0], [1, 0, 0], [0, 1, 0], [50, 0, 0], [51, 0, 0], [50, 1, 0]],
                         [[0, 1], [0, 2], [1, 2], [3, 4], [3, 5], [4, 5]], [[0, 1, 2], [3, 4, 5]])
    r = ck.ccd(s, ctx=ctx)
    assert not r.toi.collision() and r.candidate_count == 0 and r.batch_count == 1
    r = ck.ccd(plane_crossing_scene(), ctx=ctx)
    assert 0.5 - 2.0 ** -20 <= r.toi.toi <= 0.5 and r.candidate_count >= 1
    empty = scenes.SceneStep(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 2)), np.zeros((0, 3)))
    assert not ck.ccd(empty, ctx=ctx).toi.collision()


def test_resident_step_shards_union(ctx, ref):
    s = scenes.make_cloth_scene(60, 60, 0.02, 1.0, 4)
    cfg = PipelineConfig(inflation=0.01)
    rs = ck.ResidentScene(s, ctx)
    full = rs.step(cfg)
    full_pairs = rs.candidates(full.candidate_count)
    for shards in [2, 3, 8]:
        parts, tois = [], []
        for r in range(shards):
            rep = rs.step(cfg, r, shards)
            parts.append(rs.candidates(rep.candidate_count))
            tois.append(rep.toi.toi)
        union = np.concatenate(parts)
        union = union[np.lexsort((union[:, 1], union[:, 0]))]
        np.testing.assert_array_equal(union, full_pairs)
        assert min(tois) == full.toi.toi
    # determinism across repeated device runs
    again = rs.step(cfg)
    assert again.toi.toi == full.toi.toi and again.candidate_count == full.candidate_count


# ------------------------------------------------- batching, min-sep, retry

def test_batching_transparency_matches_reference(ctx, ref):
    """test_pipeline.cpp:68-87 / acceptance criterion 6: same ToI and
    candidates at every budget; batch counts and tracked bytes equal the
    reference's."""
    s = scenes.make_box_soup(30, 4.0, 0.4, 1.0, 5)
    full = ck.ccd(s, PipelineConfig(), ctx=ctx)
    assert full.batch_count == 1
    last = 1
    for budget in [1 << 22, 1 << 20, 1 << 18]:
        cfg = PipelineConfig(memory_budget=budget)
        got = ck.ccd(s, cfg, ctx=ctx)
        exp, pairs = ref.ccd(s, cfg.to_c())
        assert got.toi.toi == full.toi.toi == exp.toi
        np.testing.assert_array_equal(got.candidates, full.candidates)
        np.testing.assert_array_equal(got.candidates, pairs)
        assert got.batch_count == exp.batch_count, budget
        assert got.tracked_peak_bytes == exp.tracked_peak_bytes, budget
        assert got.batch_count >= last
        last = got.batch_count
    assert last > 1
    with pytest.raises(ck.ConfigError):
        ck.ccd(plane_crossing_scene(), PipelineConfig(memory_budget=100), ctx=ctx)


def test_query_min_separations_bit_exact(ctx, ref):
    qb = concat(scenes.random_queries(2000, seed=51), scenes.degenerate_queries(40, seed=52))
    cfg = PipelineConfig(min_sep_mode=ck.MINSEP_RELATIVE, min_sep_fraction=0.2)
    got = ck.query_min_separations(qb, cfg, ctx)
    exp = ref.query_min_separations(qb.kind, qb.points, cfg.to_c())
    assert_bits(got, exp)
    # plane-crossing scene: d0 = 1 -> 0.2 (test_pipeline.cpp:50-66)
    q = plane_crossing_query()
    assert ck.query_min_separations(q, cfg, ctx)[0] == 0.2 * 1.0
    assert ck.point_triangle_distance([0.25, 0.25, 1], [0, 0, 0], [1, 0, 0], [0, 1, 0], ctx) == 1.0


def test_relative_min_sep_pipeline(ctx, ref):
    # a colliding soup small enough for the reference: its narrow phase is
    # slow on relative-mode contacts (a 40-body soup took 3 min on 16 cores)
    s = scenes.make_box_soup(6, 3.0, 0.4, 1.0, 2)
    cfg = PipelineConfig(min_sep_mode=ck.MINSEP_RELATIVE, inflation=0.01)
    got = ck.ccd(s, cfg, ctx=ctx)
    exp, pairs = ref.ccd(s, cfg.to_c())
    assert got.toi.toi == exp.toi and got.toi.tolerance_hit == bool(exp.tolerance_hit)
    np.testing.assert_array_equal(got.candidates, pairs)
    assert exp.toi < 1.0  # the relative separations decide a real contact


def test_zero_toi_retry(ctx, ref):
    """test_pipeline.cpp:108-146: the 0.8 retry is bit-exact."""
    s = plane_crossing_scene()
    s.vertices_t0[3] = [0.25, 0.25, 1e-13]
    s.vertices_t1[3] = [0.25, 0.25, -1.0]
    cfg = PipelineConfig(narrow=NarrowConfig(no_zero_toi=True, min_separation=1e-6))
    got = ck.ccd_no_zero_toi(s, cfg, ctx=ctx)
    exp, _ = ref.ccd(s, cfg.to_c(), no_zero_retry=True)
    assert got.toi.toi == exp.toi and got.toi.zero_toi_diagnostic == bool(exp.zero_toi_diagnostic)
    assert got.toi.toi > 0.0 or got.toi.zero_toi_diagnostic
    with pytest.raises(ck.ConfigError):
        ck.ccd_no_zero_toi(s, PipelineConfig(), ctx=ctx)
    # positive plain result: no retry
    plain = ck.ccd_no_zero_toi(plane_crossing_scene(), PipelineConfig(narrow=NarrowConfig(no_zero_toi=True)), ctx=ctx)
    assert plain.toi.toi == ck.ccd(plane_crossing_scene(), ctx=ctx).toi.toi > 0
    # near-touching non-intersecting pair, Relative separation
    s2 = plane_crossing_scene()
    s2.vertices_t0[3] = [0.3, 0.3, 1e-8]
    s2.vertices_t1[3] = [0.3, 0.3, -1e-4]
    cfg2 = PipelineConfig(narrow=NarrowConfig(no_zero_toi=True), min_sep_mode=ck.MINSEP_RELATIVE)
    r2 = ck.ccd_no_zero_toi(s2, cfg2, ctx=ctx)
    e2, _ = ref.ccd(s2, cfg2.to_c(), no_zero_retry=True)
    assert r2.toi.toi == e2.toi and r2.toi.toi > 0.0


def test_query_results_fetch(ctx, ref):
    # one batch: per-query results are in the global VF-then-EE order (with
    # several broad batches the reference concatenates per-batch blocks)
    s = scenes.make_cloth_scene(20, 20, 0.02, 1.0, 7)
    cfg = PipelineConfig(inflation=0.01)
    rs = ck.ResidentScene(s, ctx)
    rep = rs.step(cfg)
    toi, flags = rs.query_results(rep.query_count)
    pairs = rs.candidates(rep.candidate_count)
    cls = ref.classify(pairs, s)
    etoi, eflags, _ = ref.narrow_phase(cls[0], cls[1], NarrowConfig().to_c())
    assert_bits(toi, etoi)
    np.testing.assert_array_equal(flags, eflags)


# ------------------------------------------------------- C5 (narrow-only batch)

def test_c5_mixed_sample_bit_exact(ctx, ref):
    """BASELINE config 5 recipe on a sample: generic queries with every
    1,000th replaced by a rotated near-degenerate (plane crossings, tangent
    double roots, parallel-above, coincident, slides) plus two slides at gap
    2e-6 that exhaust the 2^20 split budget (the config's work bombs)."""
    import os
    import oracle
    qb = concat(scenes.mixed_queries(20_000, seed=1003, every=1000, n_exhaust=0),
                scenes.degenerate_queries(2, seed=77, n_exhaust=2))
    got = ck.narrow_phase(qb, ctx=ctx)
    toi, flags, st = oracle.ref(os.cpu_count() or 1).narrow_phase(qb.kind, qb.points, NarrowConfig().to_c())
    _narrow_equal(got, toi, flags, st)
    assert (got.flags[-2:] & abi.FLAG_TOLERANCE_HIT).any()  # the VF budget bomb really exhausts


def test_c5_partition_independence(ctx):
    """Size-independent property at C5 scale: a query's result depends only
    on the query (narrowphase.hpp:93-96), so per-query ToI/flags of a 2M-query
    batch equal those of the same queries run as a small separate batch, and
    the global ToI is the min of the per-query ToIs."""
    qb = scenes.mixed_queries(2_000_000, seed=1003, every=10000, n_exhaust=4)
    big = ck.narrow_phase(qb, ctx=ctx)
    rng = np.random.default_rng(5)
    idx = np.unique(np.concatenate([rng.choice(len(qb), 4000, replace=False),
                                    np.arange(9999, len(qb), 10000)]))
    small = ck.narrow_phase(scenes.QueryBatch(qb.kind[idx], qb.points[idx]), ctx=ctx)
    assert_bits(big.toi[idx], small.toi)
    np.testing.assert_array_equal(big.flags[idx], small.flags)
    assert big.global_toi == big.toi.min()
    assert int((big.flags & abi.FLAG_TOLERANCE_HIT).astype(bool).sum()) >= 1  # a budget bomb is in the batch


# ------------------------------------------------- multi-GPU rebalance (1 GPU)

def test_rebalanced_shards_match_full_step(ctx):
    """The rebalanced multi-GPU step, simulated with two shards on one device:
    the shards' sweep keys union to the full candidate set; narrow-phasing
    equal-count slices of their concatenation (ccdk_ccd_keys_resident)
    reproduces the full step's global ToI and every query's ToI / flags."""
    import torch
    from paper_2112_06300_b200.multigpu import balanced_ranges
    s = scenes.make_cloth_scene(40, 40, 0.02, 1.0, 4)
    cfg = PipelineConfig(inflation=0.01)
    rs = ck.ResidentScene(s, ctx)
    full = rs.step(cfg)
    full_keys = None
    shard_keys = []
    for r in range(2):
        n, nb, _ = rs.broad(cfg, r, 2)
        t = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
        rs.copy_keys(t.data_ptr())
        shard_keys.append(t[:n].cpu().numpy().view(np.uint64))
    n_all, nb, _ = rs.broad(cfg, 0, 1)
    t = torch.empty(n_all, dtype=torch.int64, device="cuda")
    rs.copy_keys(t.data_ptr())
    full_keys = t.cpu().numpy().view(np.uint64)
    concat = np.concatenate(shard_keys)
    assert np.array_equal(np.sort(concat), full_keys)
    assert len(full_keys) == full.candidate_count
    # full-step per-query results, indexed by canonical key
    rs.step(cfg)
    ftoi, ffl = rs.query_results(full.query_count)
    toi = np.inf
    for lo, hi in balanced_ranges([len(k) for k in shard_keys], 2):
        sl = torch.from_numpy(concat[lo:hi].view(np.int64).copy()).cuda()
        rep = rs.narrow_keys(cfg, sl.data_ptr(), hi - lo, nb)
        toi = min(toi, rep.toi.toi)
        qt, qf = rs.query_results(rep.query_count)
        pos = np.searchsorted(full_keys, np.sort(concat[lo:hi]))
        assert_bits(qt, ftoi[pos])
        np.testing.assert_array_equal(qf, ffl[pos])
    assert toi == full.toi.toi


def test_c4_full_size_bit_exact(ctx):
    """BASELINE config 4 at full size (1,005,334 primitives) against the
    unmodified reference on all host cores: identical candidate count, and
    every query's ToI / flags bit-identical (queries in canonical order)."""
    import os
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    s = scenes.config_scene("C4")
    cfg = PipelineConfig(inflation=0.01)
    rs = ck.ResidentScene(s, ctx)
    rep = rs.step(cfg)
    got_pairs = rs.candidates(rep.candidate_count)
    toi, flags = rs.query_results(rep.query_count)
    r = oracle.ref(os.cpu_count() or 1)
    cref = PipelineConfig(inflation=0.01, broad_method=ck.BROAD_SAP, threads=os.cpu_count() or 1)
    exp, pairs = r.ccd(s, cref.to_c())
    assert rep.candidate_count == exp.candidate_count
    np.testing.assert_array_equal(got_pairs, pairs)
    assert rep.toi.toi == exp.toi
    kind, pts, _, _ = r.classify(pairs, s)
    etoi, efl, st = r.narrow_phase(kind, pts, NarrowConfig().to_c())
    assert_bits(toi, etoi)
    np.testing.assert_array_equal(flags, efl)


def test_broad_phase_quantised_filter_extremes(ctx, ref):
    """The sweep's 15-bit quantised pre-filter must stay a superset of the
    exact fp32 test whatever the coordinates: touching boxes (max == min),
    -0/+0, one huge box stretching the quantisation range, 1e30 magnitudes,
    +-FLT_MAX and infinities (round_up_reduced overflow), denormals, and a
    scene where every box is identical (zero extent)."""
    f32max = np.float32(3.4028235e38)
    cases = []
    b, s = random_boxes(77, 400)
    b.min_corner[0] = [-1e30, -1e30, -1e30]   # one box spans the whole range
    b.max_corner[0] = [1e30, 1e30, 1e30]
    cases.append((b, s))
    b, s = random_boxes(78, 300)
    b.max_corner[:, 1] = b.min_corner[:, 1]   # zero extent on one axis, touching pairs
    b.min_corner[::7] = -0.0
    b.max_corner[::7] = 0.0
    cases.append((b, s))
    b, s = random_boxes(79, 300)
    b.min_corner[:5] = -np.inf
    b.max_corner[5:10] = np.inf
    b.min_corner[10:15] = -f32max
    b.max_corner[15:20] = f32max
    cases.append((b, s))
    b, s = random_boxes(80, 200)
    b.min_corner[:] = b.min_corner[0]
    b.max_corner[:] = b.max_corner[0]
    cases.append((b, s))
    b, s = random_boxes(81, 300)
    b.min_corner *= np.float32(1e-40)         # denormal coordinates
    b.max_corner *= np.float32(1e-40)
    cases.append((b, s))
    for b, s in cases:
        for method in (abi.BROAD_STQ, abi.BROAD_SAP):
            got = ck._broad(method, b, s, None, None, ctx)
            exp, _, _ = ref.broad(method, b.as_tuple(), s)
            np.testing.assert_array_equal(got, exp)


def test_chunked_upload_equals_single_run(ctx):
    """ccdk_narrow_phase streams large batches from pinned memory in chunks
    (upload of chunk i+1 overlapping chunk i's BFS).  Results and stats —
    including the peak queue size, combined across chunks per generation —
    must equal the single-run path (same batch from pageable memory)."""
    import torch
    qb = scenes.mixed_queries(4_500_000, seed=1003, every=10000, n_exhaust=2)
    single = ck.narrow_phase(qb, ctx=ctx)  # pageable numpy -> one run
    kt = torch.from_numpy(qb.kind).pin_memory()
    pt = torch.from_numpy(qb.points).pin_memory()
    chunked = ck.narrow_phase(scenes.QueryBatch(kt.numpy(), pt.numpy()), ctx=ctx)
    assert_bits(chunked.toi, single.toi)
    np.testing.assert_array_equal(chunked.flags, single.flags)
    assert chunked.total_splits == single.total_splits
    assert chunked.evaluations == single.evaluations
    assert chunked.peak_queue == single.peak_queue
    assert chunked.generations == single.generations
    assert bits(np.array([chunked.global_toi]))[0] == bits(np.array([single.global_toi]))[0]
    # the bench's end-to-end form: pinned inputs and pinned caller-provided outputs
    toi_h = torch.empty(len(qb), dtype=torch.float64).pin_memory().numpy()
    fl_h = torch.empty(len(qb), dtype=torch.uint8).pin_memory().numpy()
    ck.narrow_phase(scenes.QueryBatch(kt.numpy(), pt.numpy()), ctx=ctx, toi_out=toi_h, flags_out=fl_h)
    assert_bits(toi_h, single.toi)
    np.testing.assert_array_equal(fl_h, single.flags)


def test_device_batch_chunking_equals_single_run(ctx):
    """ccdk_narrow_phase_device runs very large batches as consecutive BFS
    runs over chunks; outputs and stats (incl. the combined peak queue) must
    equal the host API's single run on the same queries."""
    import torch
    qb = scenes.mixed_queries(4_300_000, seed=7, every=10000, n_exhaust=1)
    single = ck.narrow_phase(qb, ctx=ctx)  # pageable numpy -> one run
    k = torch.from_numpy(qb.kind).cuda()
    p = torch.from_numpy(qb.points).cuda()
    toi = torch.empty(len(qb), dtype=torch.float64, device="cuda")
    fl = torch.empty(len(qb), dtype=torch.uint8, device="cuda")
    out = ck.narrow_phase_device(k.data_ptr(), p.data_ptr(), len(qb), toi_ptr=toi.data_ptr(),
                                 flags_ptr=fl.data_ptr(), ctx=ctx)
    assert_bits(toi.cpu().numpy(), single.toi)
    np.testing.assert_array_equal(fl.cpu().numpy(), single.flags)
    assert out.total_splits == single.total_splits and out.evaluations == single.evaluations
    assert out.peak_queue == single.peak_queue and out.generations == single.generations
    assert out.global_toi == single.global_toi


def test_concurrent_calls_share_a_context(ctx):
    """The reference's functions are reentrant and ignore `threads` (
    test_pipeline.cpp:96-106, test_narrowphase.cpp:196-211): host threads sharing one
    context get exactly the single-threaded results, including ccd's candidate pairs,
    which are fetched from the context after the step."""
    import threading
    qb = scenes.random_queries(600, seed=77)
    s1 = scenes.make_cloth_scene(16, 16, 0.02, 1.0, 3)
    s2 = scenes.make_box_soup(12, 3.0, 0.4, 1.0, 9)
    pcfg = PipelineConfig(inflation=0.01)
    exp_n = ck.narrow_phase(qb, NarrowConfig(), ctx=ctx)
    exp_c = {0: ck.ccd(s1, pcfg, ctx=ctx), 1: ck.ccd(s2, pcfg, ctx=ctx)}
    boxes = ck.build_boxes(s2, 0.01, ctx=ctx)
    exp_b = ck.stq(boxes, s2, ctx=ctx)
    errors, checked = [], []

    def work(i):
        try:
            for it in range(4):
                if (i + it) % 3 == 0:
                    got = ck.narrow_phase(qb, NarrowConfig(), threads=1 + 7 * (i % 2), ctx=ctx)
                    assert bits(got.toi).tolist() == bits(exp_n.toi).tolist()
                    assert got.flags.tolist() == exp_n.flags.tolist()
                    assert got.total_splits == exp_n.total_splits and got.peak_queue == exp_n.peak_queue
                elif (i + it) % 3 == 1:
                    k = (i + it) % 2
                    got = ck.ccd(s1 if k == 0 else s2, pcfg, ctx=ctx)
                    np.testing.assert_array_equal(got.candidates, exp_c[k].candidates)
                    assert bits(np.array([got.toi.toi]))[0] == bits(np.array([exp_c[k].toi.toi]))[0]
                else:
                    np.testing.assert_array_equal(ck.stq(boxes, s2, threads=4, ctx=ctx), exp_b)
                checked.append(1)
        except Exception as e:  # noqa: BLE001 - surfaced below
            errors.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[0]
    assert len(checked) == 16


def test_narrow_phase_caller_output_buffers(ctx):
    """Per-query results into caller-provided (here pinned) host buffers, like the C ABI's
    output pointers: identical to the returned arrays; wrong buffers are a ConfigError."""
    import torch
    qb = scenes.random_queries(2000, seed=91)
    exp = ck.narrow_phase(qb, ctx=ctx)
    toi_h = torch.full((2000,), -1.0, dtype=torch.float64).pin_memory().numpy()
    fl_h = torch.full((2000,), 255, dtype=torch.uint8).pin_memory().numpy()
    got = ck.narrow_phase(qb, ctx=ctx, toi_out=toi_h, flags_out=fl_h)
    assert np.shares_memory(got.toi, toi_h) and np.shares_memory(got.flags, fl_h)
    assert_bits(toi_h, exp.toi)
    np.testing.assert_array_equal(fl_h, exp.flags)
    assert got.total_splits == exp.total_splits and got.peak_queue == exp.peak_queue
    with pytest.raises(ck.ConfigError):
        ck.narrow_phase(qb, ctx=ctx, toi_out=np.empty(2000, np.float32))
    with pytest.raises(ck.ConfigError):
        ck.narrow_phase(qb, ctx=ctx, flags_out=np.empty(10, np.uint8))
