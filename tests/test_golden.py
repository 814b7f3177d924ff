"""Golden fixtures generated from the unmodified reference
(tests/golden/make_golden.py): the C restatement oracle must reproduce them
on CPU; the CUDA path must reproduce them on the GPU.  Bit-exact throughout."""
import json
import os

import numpy as np
import pytest

from paper_2112_06300_b200 import abi, scenes

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
G = np.load(os.path.join(HERE, "golden.npz"))
META = json.load(open(os.path.join(HERE, "golden.json")))

NARROW = {"default": dict(), "ms37": dict(max_splits=37), "sep": dict(min_separation=0.01),
          "nz": dict(no_zero_toi=True, max_splits=64)}
CCD = {"cloth20": (lambda: scenes.make_cloth_scene(20, 20, 0.02, 1.0, 1), dict(inflation=0.01)),
       "soup30_b18": (lambda: scenes.make_box_soup(30, 4.0, 0.4, 1.0, 5), dict(memory_budget=1 << 18)),
       "c1_small": (lambda: scenes.config_scene("C1", 0.02), dict(inflation=0.01))}


def b(a):
    a = np.ascontiguousarray(a)
    return a.view({8: np.uint64, 4: np.uint32, 1: np.uint8}[a.dtype.itemsize])


# ---------------------------------------------------------------- CPU: oracle

def test_oracle_rounding_and_boxes_golden(orc):
    d, u = orc.round_reduced(G["round_x"])
    np.testing.assert_array_equal(b(d), b(G["round_down"]))
    np.testing.assert_array_equal(b(u), b(G["round_up"]))
    mn, mx, kind, idx = orc.build_boxes(scenes.make_cloth_scene(9, 7, 0.02, 1.0, 3), 0.01)
    np.testing.assert_array_equal(b(mn), b(G["boxes_min"]))
    np.testing.assert_array_equal(b(mx), b(G["boxes_max"]))
    np.testing.assert_array_equal(kind, G["boxes_kind"])
    np.testing.assert_array_equal(idx, G["boxes_index"])


def test_oracle_broad_golden(orc):
    soup = scenes.make_box_soup(40, 5.0, 0.4, 1.0, 1005)
    sb = orc.build_boxes(soup, 0.01)
    pairs, rounds, mq = orc.broad(abi.BROAD_STQ, sb, soup)
    np.testing.assert_array_equal(pairs, G["soup_pairs"])
    np.testing.assert_array_equal(rounds, G["soup_rounds"])
    assert mq == META["soup_max_queue"]
    lo, _, _ = orc.broad(abi.BROAD_STQ, sb, soup, 0, META["soup_half"])
    np.testing.assert_array_equal(lo, G["soup_pairs_lo"])


@pytest.mark.parametrize("tag", sorted(NARROW))
def test_oracle_narrow_golden(orc, tag):
    toi, flags, st = orc.narrow_phase(G["q_kind"], G["q_points"], abi.narrow_cfg(**NARROW[tag]))
    np.testing.assert_array_equal(b(toi), b(G[f"narrow_{tag}_toi"]))
    np.testing.assert_array_equal(flags, G[f"narrow_{tag}_flags"])
    m = META[f"narrow_{tag}"]
    assert (st.peak_queue, st.total_splits) == (m["peak_queue"], m["total_splits"])
    assert float(st.global_toi).hex() == m["global_toi"]


def test_oracle_inclusion_golden(orc):
    for i in range(len(G["inc_boxes"])):
        r = orc.inclusion_box(G["q_kind"][i], G["q_points"][i], G["inc_boxes"][i])
        np.testing.assert_array_equal(b(r), b(G["inc_out"][i]))


@pytest.mark.parametrize("name", ["cloth20", "c1_small"])
def test_oracle_ccd_golden(orc, name):
    make, kw = CCD[name]
    rep, pairs = orc.ccd(make(), abi.pipeline_cfg(**kw))
    m = META["ccd"][name]
    np.testing.assert_array_equal(pairs, G[f"ccd_{name}_pairs"])
    assert float(rep.toi).hex() == m["toi"] and rep.query_count == m["queries"]


# ----------------------------------------------------------- GPU: CUDA path

@pytest.mark.gpu
def test_gpu_golden(ctx):
    from paper_2112_06300_b200 import ccdkit as ck
    d, u = ck.round_reduced(G["round_x"], ctx)
    np.testing.assert_array_equal(b(d), b(G["round_down"]))
    np.testing.assert_array_equal(b(u), b(G["round_up"]))
    bx = ck.build_boxes(scenes.make_cloth_scene(9, 7, 0.02, 1.0, 3), 0.01, ctx=ctx)
    np.testing.assert_array_equal(b(bx.min_corner), b(G["boxes_min"]))
    np.testing.assert_array_equal(b(bx.max_corner), b(G["boxes_max"]))
    soup = scenes.make_box_soup(40, 5.0, 0.4, 1.0, 1005)
    sb = ck.build_boxes(soup, 0.01, ctx=ctx)
    st = ck.StqStats()
    np.testing.assert_array_equal(ck.stq(sb, soup, stats=st, ctx=ctx), G["soup_pairs"])
    assert st.round_sizes == G["soup_rounds"].tolist() and st.max_queue == META["soup_max_queue"]
    q = scenes.QueryBatch(G["q_kind"], G["q_points"])
    for tag, kw in NARROW.items():
        out = ck.narrow_phase(q, ck.NarrowConfig(**kw), ctx=ctx)
        np.testing.assert_array_equal(b(out.toi), b(G[f"narrow_{tag}_toi"]))
        np.testing.assert_array_equal(out.flags, G[f"narrow_{tag}_flags"])
        m = META[f"narrow_{tag}"]
        assert (out.peak_queue, out.total_splits) == (m["peak_queue"], m["total_splits"])
    inc = ck.inclusion_boxes(G["q_kind"][:100], G["q_points"][:100], G["inc_boxes"], ctx)
    np.testing.assert_array_equal(b(inc), b(G["inc_out"]))
    for name, (make, kw) in CCD.items():
        rep = ck.ccd(make(), ck.PipelineConfig(**kw), ctx=ctx)
        m = META["ccd"][name]
        np.testing.assert_array_equal(rep.candidates, G[f"ccd_{name}_pairs"])
        assert float(rep.toi.toi).hex() == m["toi"]
        assert (rep.query_count, rep.batch_count, rep.tracked_peak_bytes) == \
            (m["queries"], m["batch_count"], m["tracked_peak_bytes"])
