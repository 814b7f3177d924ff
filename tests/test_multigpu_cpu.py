"""Multi-GPU host logic on CPU: world_size 2 over gloo.

Each rank sweeps its equal-work slice of sorted left positions (the device
partition rule, restated in multigpu.shard_bounds), runs classify + narrow on
its own candidates with the CPU checker standing in for the device, and the
ranks combine the ToI with the single allreduce(min).  The union of the
shards' candidate sets must equal the single-process set, and the reduced ToI
the single-process ToI (the SweepRange contract, broadphase.hpp:37-43).
"""
import os
import socket

import numpy as np
import pytest

from paper_2112_06300_b200 import abi, scenes
from paper_2112_06300_b200.multigpu import shard_bounds, sorted_run_lengths


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2112_06300_b200.multigpu import allreduce_min_toi

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = oracle.orc()
    s = scenes.make_cloth_scene(24, 24, 0.02, 1.0, 4)
    boxes = orc.build_boxes(s, 0.01)
    k = len(boxes[0])
    axis = orc.choose_axis(boxes[0], boxes[1])
    _, run_len = sorted_run_lengths(boxes[0], boxes[1], axis)
    lo, hi = shard_bounds(run_len, 0, k - 1, rank, world)
    pairs, _, _ = orc.broad(abi.BROAD_STQ, boxes, s, lo, hi)
    kind, pts, _, _ = orc.classify(pairs, s)
    toi = np.inf
    if len(kind):
        t, _, st = orc.narrow_phase(kind, pts, abi.narrow_cfg())
        toi = st.global_toi
    tt = torch.tensor([toi], dtype=torch.float64)
    allreduce_min_toi(tt)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([len(pairs)], dtype=torch.int64))
    mx = int(max(x.item() for x in sizes))
    buf = torch.zeros((mx, 2), dtype=torch.int64)
    buf[:len(pairs)] = torch.from_numpy(pairs.astype(np.int64))
    gathered = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf)
    if rank == 0:
        union = np.concatenate([g[:int(n.item())].numpy() for g, n in zip(gathered, sizes)]).astype(np.uint64)
        np.savez(result_path, union=union, toi=tt.numpy(), work=np.array([int(run_len[lo:hi].sum())]))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_step_union_and_min_toi(tmp_path):
    import torch.multiprocessing as mp

    import oracle
    world = 2
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = np.load(out)
    s = scenes.make_cloth_scene(24, 24, 0.02, 1.0, 4)
    rep, pairs = oracle.orc().ccd(s, abi.pipeline_cfg(inflation=0.01))
    union = res["union"]
    union = union[np.lexsort((union[:, 1], union[:, 0]))]
    np.testing.assert_array_equal(union, pairs)
    assert res["toi"][0] == rep.toi


@pytest.mark.parametrize("count", [1, 2, 3, 8])
def test_shard_bounds_partition(count):
    rng = np.random.default_rng(5)
    run_len = rng.integers(0, 50, size=1000).astype(np.uint64)
    run_len[[3, 500]] = 100000  # heavy rows
    bounds = [shard_bounds(run_len, 10, 990, r, count) for r in range(count)]
    assert bounds[0][0] == 10 and bounds[-1][1] == 990
    for a, b in zip(bounds, bounds[1:]):
        assert a[1] == b[0]
    total = int(run_len[10:990].sum())
    for lo, hi in bounds:  # every shard's work is within one row of the ideal share
        assert int(run_len[lo:hi].sum()) <= total / count + int(run_len.max())


def _rebalance_worker(rank, world, port, result_path, policy="contiguous"):
    import torch
    import torch.distributed as dist

    from paper_2112_06300_b200.multigpu import balanced_ranges, rebalance_keys

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    counts = [37, 5] if world == 2 else [1] * world
    rng = np.random.default_rng(100 + rank)
    keys = torch.from_numpy(rng.integers(0, 1 << 40, counts[rank], dtype=np.int64))
    mine = rebalance_keys(keys, counts, rank, world, policy=policy)
    # what every rank holds, gathered for the check
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([mine.numel()], dtype=torch.int64))
    mx = max(int(x.item()) for x in sizes)
    buf = torch.zeros(mx, dtype=torch.int64)
    buf[:mine.numel()] = mine
    got = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(got, buf)
    src = [torch.zeros(max(counts), dtype=torch.int64) for _ in range(world)]
    pad = torch.zeros(max(counts), dtype=torch.int64)
    pad[:keys.numel()] = keys
    dist.all_gather(src, pad)
    if rank == 0:
        concat = np.concatenate([s[:c].numpy() for s, c in zip(src, counts)])
        held = [g[:int(n.item())].numpy() for g, n in zip(got, sizes)]
        if policy == "contiguous":
            rngs = balanced_ranges(counts, world)
            ok = all(np.array_equal(h, concat[lo:hi]) for h, (lo, hi) in zip(held, rngs))
        else:  # rank r holds global indices r, r+N, r+2N, ... in order
            ok = all(np.array_equal(h, concat[r::world]) for r, h in enumerate(held))
        ok = ok and max(len(h) for h in held) - min(len(h) for h in held) <= 1
        with open(result_path, "w") as f:
            f.write("ok" if ok else "bad")
    dist.destroy_process_group()


@pytest.mark.parametrize("policy", ["interleave", "contiguous"])
def test_rebalance_keys_gloo_world2(tmp_path, policy):
    """after the sweep, one all_to_all moves pair keys so each
    rank holds an equal share (within one) of the rank-ordered concatenation:
    every N-th candidate (interleave, the default) or a contiguous slice."""
    import torch.multiprocessing as mp
    out = tmp_path / "res.txt"
    mp.start_processes(_rebalance_worker, args=(2, _free_port(), str(out), policy), nprocs=2, join=True,
                       start_method="spawn")
    assert out.read_text() == "ok"


def test_interleave_splits_host():
    from paper_2112_06300_b200.multigpu import interleave_splits
    counts = [10, 3, 7, 0, 5]
    world = 5
    total = sum(counts)
    sends = [interleave_splits(counts, r, world)[0] for r in range(world)]
    recvs = [interleave_splits(counts, r, world)[1] for r in range(world)]
    for r in range(world):
        assert sum(sends[r]) == counts[r]
        assert sum(recvs[r]) == len(range(r, total, world))
        for s in range(world):
            assert sends[s][r] == recvs[r][s]


def test_exchange_splits_host():
    from paper_2112_06300_b200.multigpu import balanced_ranges, exchange_splits
    counts = [10, 3, 7, 0]
    rng = balanced_ranges(counts, 4)
    assert [hi - lo for lo, hi in rng] == [5, 5, 5, 5]
    sends = [exchange_splits(counts, r, 4)[0] for r in range(4)]
    recvs = [exchange_splits(counts, r, 4)[1] for r in range(4)]
    for r in range(4):
        assert sum(sends[r]) == counts[r]
        assert sum(recvs[r]) == rng[r][1] - rng[r][0]
        for s in range(4):
            assert sends[s][r] == recvs[r][s]
