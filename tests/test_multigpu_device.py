"""The multi-GPU host layer through the REAL device calls at world size 2.

The build and test boxes have one GPU, and NCCL refuses two ranks on one
device, so the two ranks share cuda:0 (one ccdk context each) and talk over
gloo with device tensors staged through the host (multigpu.host_staged).
Every ccdk call is the one a rank of an N-GPU job makes: the resident scene,
ccdk_ccd_resident on a SweepRange shard (ShardedCcd), and the split step of
RebalancedCcd — ccdk_broad_resident, all_gather of the counts, all_to_all of
the 8-byte pair keys, ccdk_ccd_keys_resident on the balanced slice,
ccdk_copy_last_toi + allreduce(min).  Checked against the single-process
C restatement (oracle/liborc): the shards' candidate sets partition the full
set, the balanced slices' query counts add up, and both steps reduce to the
single-process global ToI.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


SCENE = dict(nx=40, ny=40, jitter=0.02, drop=1.0, seed=4)


def _worker(rank, world, port, out_dir, slab="auto"):
    import torch
    import torch.distributed as dist

    if slab != "auto":
        os.environ["CCDK_SLAB"] = slab  # force the slab-mode sweep (shards over entry rows)

    from paper_2112_06300_b200 import ccdkit as ck, native, scenes
    from paper_2112_06300_b200.multigpu import RebalancedCcd, ShardedCcd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    s = scenes.make_cloth_scene(SCENE["nx"], SCENE["ny"], SCENE["jitter"], SCENE["drop"], SCENE["seed"])
    cfg = ck.PipelineConfig(inflation=0.01)
    ctx = native.Context(0)
    resident = ck.ResidentScene(s, ctx)

    sharded = ShardedCcd(resident, rank, world)
    rep = sharded.step(cfg)
    toi_sharded = sharded.global_toi(rep)
    mine = resident.candidates(rep.candidate_count).astype(np.int64).reshape(-1, 2)

    rebal = RebalancedCcd(resident, rank, world)
    rep2 = rebal.step(cfg)
    toi_rebal = rebal.global_toi(rep2)

    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([len(mine)], dtype=torch.int64))
    mx = max(1, int(max(x.item() for x in sizes)))
    buf = torch.zeros((mx, 2), dtype=torch.int64)
    buf[:len(mine)] = torch.from_numpy(mine)
    gathered = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf)
    nq = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(nq, torch.tensor([rep2.query_count], dtype=torch.int64))
    if rank == 0:
        union = np.concatenate([g[:int(n.item())].numpy() for g, n in zip(gathered, sizes)])
        np.savez(os.path.join(out_dir, "res.npz"), union=union.astype(np.uint64),
                 toi=np.array([toi_sharded, toi_rebal]), shard_sizes=np.array([int(x.item()) for x in sizes]),
                 balanced_queries=np.array([int(x.item()) for x in nq]),
                 counts=np.array(rep2.shard_counts))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("slab", ["auto", "1"])
def test_world2_on_one_device_matches_single_process(tmp_path, slab):
    import torch.multiprocessing as mp

    import oracle
    from paper_2112_06300_b200 import abi, scenes

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), slab), nprocs=2, join=True)
    res = np.load(tmp_path / "res.npz")
    s = scenes.make_cloth_scene(SCENE["nx"], SCENE["ny"], SCENE["jitter"], SCENE["drop"], SCENE["seed"])
    rep, pairs = oracle.orc().ccd(s, abi.pipeline_cfg(inflation=0.01))
    union = res["union"]
    union = union[np.lexsort((union[:, 1], union[:, 0]))]
    np.testing.assert_array_equal(union, pairs)           # shards partition the candidate set
    assert all(n > 0 for n in res["shard_sizes"])         # both ranks swept real work
    assert int(res["balanced_queries"].sum()) == len(pairs)
    assert abs(int(res["balanced_queries"][0]) - int(res["balanced_queries"][1])) <= 1
    assert int(res["counts"].sum()) == len(pairs)
    assert res["toi"][0] == rep.toi and res["toi"][1] == rep.toi
