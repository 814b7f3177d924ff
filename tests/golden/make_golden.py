"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz (+ golden.json for scalars).  Needs
oracle/_ref/libccdref.so, i.e. a machine with /root/reference; the committed
fixtures let the oracle restatement and the GPU path be checked anywhere.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from paper_2112_06300_b200 import abi, scenes  # noqa: E402
from fixtures import random_subboxes, special_doubles  # noqa: E402


def main():
    R = oracle.ref()
    out, meta = {}, {}
    x = special_doubles(11, 4000)
    d, u = R.round_reduced(x)
    out.update(round_x=x, round_down=d, round_up=u)

    cloth = scenes.make_cloth_scene(9, 7, 0.02, 1.0, 3)
    mn, mx, kind, idx = R.build_boxes(cloth, 0.01)
    out.update(boxes_min=mn, boxes_max=mx, boxes_kind=kind, boxes_index=idx)

    soup = scenes.make_box_soup(40, 5.0, 0.4, 1.0, 1005)
    sb = R.build_boxes(soup, 0.01)
    pairs, rounds, mq = R.broad(abi.BROAD_STQ, sb, soup)
    out.update(soup_pairs=pairs, soup_rounds=rounds)
    meta["soup_max_queue"] = int(mq)
    half = len(sb[0]) // 2
    pairs_lo, _, _ = R.broad(abi.BROAD_STQ, sb, soup, 0, half)
    out.update(soup_pairs_lo=pairs_lo)
    meta["soup_half"] = half

    q = scenes.random_queries(400, seed=1003)
    out.update(q_kind=q.kind, q_points=q.points)
    for tag, cfg in [("default", abi.narrow_cfg()), ("ms37", abi.narrow_cfg(max_splits=37)),
                     ("sep", abi.narrow_cfg(min_separation=0.01)), ("nz", abi.narrow_cfg(no_zero_toi=1, max_splits=64))]:
        toi, flags, st = R.narrow_phase(q.kind, q.points, cfg)
        out[f"narrow_{tag}_toi"] = toi
        out[f"narrow_{tag}_flags"] = flags
        meta[f"narrow_{tag}"] = {"peak_queue": int(st.peak_queue), "total_splits": int(st.total_splits),
                                 "global_toi": float(st.global_toi).hex()}

    boxes, _ = random_subboxes(77, 100)
    inc = np.stack([R.inclusion_box(q.kind[i], q.points[i], boxes[i]) for i in range(100)])
    out.update(inc_boxes=boxes, inc_out=inc)

    meta["ccd"] = {}
    for name, s, cfg in [("cloth20", scenes.make_cloth_scene(20, 20, 0.02, 1.0, 1), abi.pipeline_cfg(inflation=0.01)),
                         ("soup30_b18", scenes.make_box_soup(30, 4.0, 0.4, 1.0, 5), abi.pipeline_cfg(memory_budget=1 << 18)),
                         ("c1_small", scenes.config_scene("C1", 0.02), abi.pipeline_cfg(inflation=0.01))]:
        rep, p = R.ccd(s, cfg)
        out[f"ccd_{name}_pairs"] = p
        meta["ccd"][name] = {"toi": float(rep.toi).hex(), "candidates": int(rep.candidate_count),
                             "queries": int(rep.query_count), "batch_count": int(rep.batch_count),
                             "tracked_peak_bytes": int(rep.tracked_peak_bytes),
                             "tolerance_hit": int(rep.tolerance_hit)}
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", sorted(out))


if __name__ == "__main__":
    main()
