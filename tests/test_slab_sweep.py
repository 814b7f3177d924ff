"""Slab-mode sweep (K5', ccdk_broad.cu) against the reference.

The full-range broad phase (ccd's default step, stq/sap without StqStats or
SweepRange) sweeps per slab of a second axis and emits every pair only in
its canonical slab.  By default it runs from 200k boxes on; CCDK_SLAB=1
forces it (read per call), so every case here runs BOTH sweeps on the same
boxes and compares each with the reference's candidate set bit for bit
(broadphase.cpp:69-127): cloth, box soups, the n-body config with 20x bodies
and walls, un-jittered grids (exact ties along the sweep and slab axes),
point-sized boxes, a single-slab scene (no second axis to cut: falls back),
arbitrary box lists through the general API, and a C4 step.
"""
import os

import numpy as np
import pytest

from paper_2112_06300_b200 import abi, ccdkit as ck, scenes

pytestmark = pytest.mark.gpu


class _Slab:
    def __init__(self, value):
        self.value = value

    def __enter__(self):
        self.old = os.environ.get("CCDK_SLAB")
        os.environ["CCDK_SLAB"] = self.value

    def __exit__(self, *a):
        if self.old is None:
            os.environ.pop("CCDK_SLAB", None)
        else:
            os.environ["CCDK_SLAB"] = self.old


def _scenes():
    flat = scenes.make_cloth_scene(50, 2, 0.0, 1.0, 3)  # a strip: one slab only
    return [scenes.make_cloth_scene(40, 40, 0.02, 1.0, 1),
            scenes.make_cloth_scene(64, 64, 0.0, 1.0, 2),   # exact ties everywhere
            scenes.make_cloth_scene(30, 90, 0.0, 2.5, 7),
            scenes.make_box_soup(300, 8.0, 0.45, 0.9, 42),
            scenes.make_box_soup(2000, 20.0, 0.3, 1.5, 11),
            scenes.config_scene("C1", 0.2),
            scenes.config_scene("C3", 0.02),
            flat]


@pytest.mark.parametrize("idx", range(8))
def test_slab_and_1d_sweeps_equal_reference(ctx, ref, idx):
    s = _scenes()[idx]
    for infl in (0.0, 0.01):
        b = ck.build_boxes(s, infl, ctx=ctx)
        exp, _, _ = ref.broad(abi.BROAD_STQ, b.as_tuple(), s)
        for mode in ("1", "0"):
            with _Slab(mode):
                got = ck.stq(b, s, ctx=ctx)
                np.testing.assert_array_equal(got, exp, err_msg=f"CCDK_SLAB={mode} inflation={infl}")
                got_sap = ck.sap(b, s, ctx=ctx)
                np.testing.assert_array_equal(got_sap, exp)


def test_slab_mode_point_boxes_and_arbitrary_lists(ctx, ref):
    """Zero-extent boxes (static vertices, inflation 0) and a box list that is
    not a scene's build order (random owners), through the general API."""
    rng = np.random.default_rng(5)
    s = scenes.make_box_soup(400, 10.0, 0.4, 0.0, 3)  # motion 0: static, many degenerate extents
    b = ck.build_boxes(s, 0.0, ctx=ctx)
    perm = rng.permutation(len(b.owner_kind))
    shuffled = ck.Boxes(b.min_corner[perm], b.max_corner[perm], b.owner_kind[perm], b.owner_index[perm])
    exp, _, _ = ref.broad(abi.BROAD_STQ, shuffled.as_tuple(), s)
    for mode in ("1", "0"):
        with _Slab(mode):
            np.testing.assert_array_equal(ck.stq(shuffled, s, ctx=ctx), exp)


def test_slab_mode_runs_on_a_full_step(ctx, ref):
    """The default C4-size path takes slab mode; the step's candidates and
    ToI equal the reference's."""
    s = scenes.make_cloth_scene(200, 200, 0.02, 1.0, 4)  # ~240k boxes: above the slab threshold
    cfg = ck.PipelineConfig(inflation=0.01)
    rep = ck.ccd(s, cfg, ctx=ctx)
    assert rep.device["sweep_slabs"] > 1 and rep.device["sweep_entries"] >= s.primitive_count()
    exp, pairs = ref.ccd(s, cfg.to_c())
    np.testing.assert_array_equal(rep.candidates, pairs)
    assert rep.toi.toi == exp.toi
    with _Slab("0"):
        rep1 = ck.ccd(s, cfg, ctx=ctx)
    assert rep1.device["sweep_slabs"] == 0
    np.testing.assert_array_equal(rep1.candidates, pairs)


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_slab_mode_shards_partition_the_set(ctx, ref, shards):
    """Multi-GPU broad phase in slab mode: rank r sweeps the entry rows that
    split the total window length evenly; the shards' keys are disjoint and
    union to the full candidate set."""
    import torch
    s = scenes.make_box_soup(2500, 22.0, 0.35, 1.2, 17)
    cfg = ck.PipelineConfig(inflation=0.01)
    rs = ck.ResidentScene(s, ctx)
    with _Slab("1"):
        n_all, nb, _ = rs.broad(cfg, 0, 1)
        t = torch.empty(max(n_all, 1), dtype=torch.int64, device="cuda")
        rs.copy_keys(t.data_ptr())
        full = np.sort(t[:n_all].cpu().numpy().view(np.uint64))
        parts = []
        for r in range(shards):
            n, nb2, _ = rs.broad(cfg, r, shards)
            assert nb2 == nb
            t = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
            rs.copy_keys(t.data_ptr())
            parts.append(t[:n].cpu().numpy().view(np.uint64))
        rep = rs.step(cfg)
        assert rep.device["sweep_slabs"] > 1
    concat = np.concatenate(parts)
    assert len(np.unique(concat)) == len(concat)  # disjoint
    np.testing.assert_array_equal(np.sort(concat), full)
    b = ck.build_boxes(s, 0.01, ctx=ctx)
    exp, _, _ = ref.broad(abi.BROAD_STQ, b.as_tuple(), s)
    assert len(full) == len(exp)
