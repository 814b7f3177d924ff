"""run_batched on a caller's box list (ccdk_run_batched) against the reference.

pipeline.cpp:179-215 batches ANY box list: the broad phase sweeps the given
boxes (broadphase.cpp, ties by owner), halves SweepRange ranges while the
candidates exceed the budget's pair capacity — sorted positions for stq/sap,
raw box positions for bf (pipeline.cpp:65-77, 140-159) — and then classifies
and narrows each broad batch.  Checked bit for bit against the reference
library (oracle/_ref) on: the scene's own boxes shuffled, a subset of the
primitives, duplicated owners, boxes inflated differently from any
cfg.inflation, small budgets under all three methods (the batch counts
differ between bf and stq), the empty list, and the owner range check.
"""
import numpy as np
import pytest

from paper_2112_06300_b200 import abi, ccdkit as ck, native, scenes

pytestmark = pytest.mark.gpu


def _own_boxes(s, infl, ctx):
    return ck.build_boxes(s, infl, ctx=ctx)


def _check(ctx, ref, s, boxes, cfg):
    exp, pairs, bb, nb = ref.run_batched(s, boxes.as_tuple(), cfg.to_c())
    trace = ck.BatchTrace()
    rep = ck.CcdReport(ck.ToiResult(), 0, 0, 0, {"CB": 0.5}, 0, None)
    toi = ck.run_batched(s, boxes, cfg, trace, rep, ctx=ctx)
    np.testing.assert_array_equal(rep.candidates.reshape(-1, 2), pairs)
    assert toi.toi == exp.toi and rep.toi.toi == exp.toi
    assert toi.tolerance_hit == bool(exp.tolerance_hit)
    assert toi.zero_toi_diagnostic == bool(exp.zero_toi_diagnostic)
    assert rep.candidate_count == exp.candidate_count and rep.query_count == exp.query_count
    assert (trace.broad_batches, trace.narrow_batches) == (bb, nb)
    assert rep.batch_count == exp.batch_count
    assert rep.tracked_peak_bytes == exp.tracked_peak_bytes
    assert rep.per_stage_times["CB"] == 0.5  # run_batched leaves CB alone
    return trace


@pytest.mark.parametrize("method", [abi.BROAD_STQ, abi.BROAD_BF, abi.BROAD_SAP])
def test_shuffled_own_boxes(ctx, ref, method):
    s = scenes.make_cloth_scene(24, 24, 0.02, 1.0, 3)
    b = _own_boxes(s, 0.01, ctx)
    perm = np.random.default_rng(1).permutation(len(b))
    shuffled = ck.Boxes(b.min_corner[perm], b.max_corner[perm], b.owner_kind[perm], b.owner_index[perm])
    _check(ctx, ref, s, shuffled, ck.PipelineConfig(inflation=0.01, broad_method=method))


@pytest.mark.parametrize("method", [abi.BROAD_STQ, abi.BROAD_BF, abi.BROAD_SAP])
@pytest.mark.parametrize("budget", [1 << 19, 3 << 18, 1 << 20])
def test_small_budgets_batch_like_the_reference(ctx, ref, method, budget):
    """Range halving: bf splits raw positions, stq/sap sorted positions, so
    the broad/narrow batch counts depend on the method and the box order."""
    s = scenes.make_cloth_scene(24, 24, 0.02, 1.0, 5)
    b = _own_boxes(s, 0.01, ctx)
    perm = np.random.default_rng(budget).permutation(len(b))
    shuffled = ck.Boxes(b.min_corner[perm], b.max_corner[perm], b.owner_kind[perm], b.owner_index[perm])
    cfg = ck.PipelineConfig(inflation=0.01, broad_method=method, memory_budget=budget)
    t = _check(ctx, ref, s, shuffled, cfg)
    assert t.broad_batches > 1


def test_subset_and_duplicate_owners(ctx, ref):
    s = scenes.make_box_soup(300, 8.0, 0.45, 0.9, 42)
    b = _own_boxes(s, 0.0, ctx)
    rng = np.random.default_rng(7)
    keep = np.sort(rng.choice(len(b), size=len(b) * 2 // 3, replace=False))
    dup = rng.choice(keep, size=len(keep) // 4)
    sel = np.concatenate([keep, dup])
    rng.shuffle(sel)
    # duplicates get distinct (wider) boxes: the same owner under two boxes
    mn = b.min_corner[sel].copy()
    mx = b.max_corner[sel].copy()
    mx[len(keep):] += np.float32(0.05)
    boxes = ck.Boxes(mn, mx, b.owner_kind[sel], b.owner_index[sel])
    for method in (abi.BROAD_STQ, abi.BROAD_BF):
        _check(ctx, ref, s, boxes, ck.PipelineConfig(broad_method=method))
        _check(ctx, ref, s, boxes, ck.PipelineConfig(broad_method=method, memory_budget=1 << 19))


def test_boxes_not_from_any_inflation(ctx, ref):
    """Custom boxes (per-primitive random padding): cfg.inflation plays no
    part, the candidates are the overlaps of the given boxes."""
    s = scenes.make_cloth_scene(30, 30, 0.02, 1.0, 9)
    b = _own_boxes(s, 0.0, ctx)
    pad = np.random.default_rng(3).uniform(0, 0.03, size=(len(b), 1)).astype(np.float32)
    boxes = ck.Boxes(b.min_corner - pad, b.max_corner + pad, b.owner_kind, b.owner_index)
    _check(ctx, ref, s, boxes, ck.PipelineConfig(inflation=0.5))
    # Relative mode (per-query separations, classify not fused); the
    # reference's narrow phase is very slow on relative-mode contacts, so the
    # scene is a small soup whose padded candidates do not collide
    s = scenes.make_box_soup(5, 3.0, 0.4, 1.0, 6)
    b = _own_boxes(s, 0.0, ctx)
    pad = np.random.default_rng(4).uniform(0, 0.02, size=(len(b), 1)).astype(np.float32)
    boxes = ck.Boxes(b.min_corner - pad, b.max_corner + pad, b.owner_kind, b.owner_index)
    _check(ctx, ref, s, boxes, ck.PipelineConfig(min_sep_mode=abi.MINSEP_RELATIVE))


def test_large_list_takes_the_slab_sweep(ctx, ref):
    s = scenes.make_cloth_scene(200, 200, 0.02, 1.0, 4)  # ~240k boxes
    b = _own_boxes(s, 0.01, ctx)
    perm = np.random.default_rng(11).permutation(len(b))
    boxes = ck.Boxes(b.min_corner[perm], b.max_corner[perm], b.owner_kind[perm], b.owner_index[perm])
    _check(ctx, ref, s, boxes, ck.PipelineConfig(inflation=0.01))


def test_empty_list_and_bad_owners(ctx, ref):
    s = scenes.make_cloth_scene(8, 8, 0.02, 1.0, 2)
    empty = ck.Boxes(np.zeros((0, 3), np.float32), np.zeros((0, 3), np.float32), np.zeros(0, np.uint8),
                     np.zeros(0, np.uint32))
    t = _check(ctx, ref, s, empty, ck.PipelineConfig())
    assert (t.broad_batches, t.narrow_batches) == (0, 1)
    b = _own_boxes(s, 0.0, ctx)
    for kind, index in ((abi.KIND_VERTEX, s.nv), (abi.KIND_EDGE, s.ne), (abi.KIND_FACE, s.nf + 3)):
        idx = b.owner_index.copy()
        sel = np.flatnonzero(b.owner_kind == kind)[0]
        idx[sel] = index
        bad = ck.Boxes(b.min_corner, b.max_corner, b.owner_kind, idx)
        with pytest.raises(native.InvalidInput, match="owner index out of range"):
            ck.run_batched(s, bad, ck.PipelineConfig(), ck.BatchTrace(), ctx=ctx)
    # the context stays usable
    _check(ctx, ref, s, b, ck.PipelineConfig())


def test_trace_accumulates_across_calls(ctx):
    s = scenes.make_cloth_scene(16, 16, 0.02, 1.0, 2)
    b = _own_boxes(s, 0.01, ctx)
    t = ck.BatchTrace()
    rep = ck.CcdReport(ck.ToiResult(), 0, 0, 0, {}, 0, None)
    cfg = ck.PipelineConfig(inflation=0.01)
    ck.run_batched(s, b, cfg, t, rep, ctx=ctx)
    ck.run_batched(s, b, cfg, t, rep, ctx=ctx)
    assert (t.broad_batches, t.narrow_batches) == (2, 2)
    assert rep.batch_count == 2  # max(1, trace.narrow_batches), as pipeline.cpp:202
    full = ck.ccd(s, cfg, ctx=ctx)
    np.testing.assert_array_equal(rep.candidates, full.candidates)
    assert rep.toi.toi == full.toi.toi
