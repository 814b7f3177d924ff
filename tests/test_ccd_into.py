"""ccdk_ccd_into's candidate-sink contract (include/ccdk.h), through ctypes.

The drop-in's ccdkit::ccd returns CcdReport::candidates (pipeline.cpp:209)
through this entry: the sink is called first with pairs == NULL and the
count, then with the canonical list in CandidatePair layout ({u8 kind, 3 zero
bytes, u32 index} x 2 per pair) — on a worker thread overlapping the narrow
phase for single-batch steps, inline at the end for budget-batched ones.
Checked: the list equals ccdk_ccd + ccdk_fetch_pairs and the reference's,
the call order, the empty-scene case, the batched path, and a failing sink.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2112_06300_b200 import abi, ccdkit as ck, native, scenes

pytestmark = pytest.mark.gpu

SINK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_uint64)


def _into(ctx, s, cfg, fail=False):
    calls = []

    def sink(user, pairs, n):
        if not pairs:
            calls.append(("count", n))
            return 1 if fail else 0
        raw = np.ctypeslib.as_array(pairs, shape=(2 * n,)).copy() if n else np.empty(0, np.uint64)
        calls.append(("data", n, raw))
        return 0

    cb = SINK(sink)
    r = abi.Report()
    rc = native.lib().ccdk_ccd_into(ctx.h, native.p(s.vertices_t0, native.P_F64), native.p(s.vertices_t1, native.P_F64),
                                    s.nv, native.p(s.edges, native.P_U32), s.ne, native.p(s.faces, native.P_U32), s.nf,
                                    C.byref(cfg.to_c()), C.byref(r), cb, None)
    return rc, r, calls


def _as_packed(raw):
    """CandidatePair layout (kind | index << 32 per id) -> C-ABI ids ((kind << 32) | index)."""
    ids = (raw >> np.uint64(32)) | ((raw & np.uint64(0xFF)) << np.uint64(32))
    return ids.reshape(-1, 2)


@pytest.mark.parametrize("budget", [None, 2 << 20])
def test_sink_receives_the_canonical_list(ctx, ref, budget):
    s = scenes.make_cloth_scene(48, 48, 0.02, 1.0, 5)
    cfg = ck.PipelineConfig(inflation=0.01) if budget is None else ck.PipelineConfig(inflation=0.01,
                                                                                    memory_budget=budget)
    rc, r, calls = _into(ctx, s, cfg)
    assert rc == 0, native.lib().ccdk_last_error()
    assert [c[0] for c in calls] == ["count", "data"]
    assert calls[0][1] == calls[1][1] == r.candidate_count
    raw = calls[1][2]
    # padding bytes are zero, kinds are 0..2
    assert np.all((raw & np.uint64(0xFFFFFF00)) == 0) and np.all((raw & np.uint64(0xFF)) <= 2)
    exp, pairs = ref.ccd(s, cfg.to_c())
    np.testing.assert_array_equal(_as_packed(raw), pairs)
    assert r.toi == exp.toi and r.batch_count == exp.batch_count
    if budget is not None:
        assert r.batch_count > 1 or r.broad_batches > 1  # the batched (inline) export path ran


def test_sink_on_an_empty_candidate_set(ctx):
    s = scenes.SceneStep(np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]]), np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]]),
                         np.zeros((0, 2), np.uint32), np.array([[0, 1, 2]], np.uint32))
    rc, r, calls = _into(ctx, s, ck.PipelineConfig(inflation=0.01))
    assert rc == 0 and r.candidate_count == 0
    assert [c[:2] for c in calls] == [("count", 0), ("data", 0)]


def test_failing_sink_fails_the_call_without_a_second_call(ctx):
    s = scenes.make_cloth_scene(16, 16, 0.02, 1.0, 2)
    rc, r, calls = _into(ctx, s, ck.PipelineConfig(inflation=0.01), fail=True)
    assert rc == abi.OOM
    assert [c[0] for c in calls] == ["count"]
    # the context stays usable
    rc, r, calls = _into(ctx, s, ck.PipelineConfig(inflation=0.01))
    assert rc == 0 and [c[0] for c in calls] == ["count", "data"]
