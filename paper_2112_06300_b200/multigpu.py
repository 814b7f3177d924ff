"""Multi-GPU host layer: one process per GPU, sweep start-ranges partitioned
across ranks, global min-ToI combined with ONE allreduce(min).

SURVEY §8(e): every rank holds the replicated scene, builds and sorts the
full box array (~0.1 ms at 1M boxes), computes run lengths, and sweeps only
its slice of sorted left positions — the slices split the total pair-test
work (sum of run lengths) evenly, which is the reference's SweepRange
contract (broadphase.hpp:37-43: the union over a partition equals the full
candidate set).  Candidate sets are disjoint by construction (a pair is
emitted by its lower sorted position), so the data path needs no collective;
the only exchange is the 8-byte allreduce(min) of the ToI, run on the device
buffer the step wrote (NCCL over NVLink on GPUs, gloo in the CPU tests).

Narrow-phase load balance: equal sweep work does not mean
equal narrow work, so RebalancedCcd splits the step at the candidate list:
after the sweep, ranks all-gather their counts (N integers) and move pair
keys with ONE all_to_all so that rank r narrow-phases every N-th candidate
(global index = r mod N) of the rank-ordered concatenation — interleaved,
because per-query BFS cost is clustered along the canonical order (see
rebalance_keys).  Every rank holds
the replicated scene, so an 8-byte key is all a rank needs to gather the
query's coordinates; per-query results are partition-independent
(narrowphase.hpp:93-96), so the ToI is unchanged.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(run_len: np.ndarray, lo: int, hi: int, rank: int, count: int) -> tuple[int, int]:
    """Host restatement of the device partition (ccdk_broad.cu k_shard_range):
    shard r covers sorted left positions [B_r, B_{r+1}) where B_r is the first
    p in [lo, hi) whose exclusive prefix of run lengths reaches floor(W*r/S)."""
    incl = np.cumsum(run_len.astype(np.uint64))
    W = int(incl[hi - 1]) if hi > lo else 0

    def boundary(r):
        if r == 0:
            return lo
        if r >= count:
            return hi
        T = (W // count) * r + ((W % count) * r) // count
        a, b = lo, hi
        while a < b:
            m = (a + b) >> 1
            e = 0 if m == lo else int(incl[m - 1])
            if e >= T:
                b = m
            else:
                a = m + 1
        return a

    return boundary(rank), boundary(rank + 1)


def sorted_run_lengths(min_corner: np.ndarray, max_corner: np.ndarray, axis: int) -> tuple[np.ndarray, np.ndarray]:
    """(order, run_len) of the sweep along `axis`: order sorts by min (ties by
    slot, -0 == +0), run_len[p] = #{j > p : min[j] <= max[p]} (STQ rounds)."""
    mn = min_corner[:, axis].astype(np.float32)
    key = mn.copy()
    key[key == 0] = 0.0  # -0 -> +0
    order = np.lexsort((np.arange(mn.size), key))
    smin = mn[order]
    smax = max_corner[order, axis].astype(np.float32)
    end = np.searchsorted(smin, smax, side="right")
    p = np.arange(mn.size)
    end = np.maximum(end, p + 1)
    return order, (end - p - 1).astype(np.uint64)


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: the legacy default stream, torch's stream 0


def host_staged(group=None) -> bool:
    """gloo moves host memory: device tensors are staged through the host
    (the world-2-on-one-GPU tests; NCCL refuses two ranks on one device).
    Under NCCL every collective runs on the device buffers directly."""
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def allreduce_min_toi(toi_tensor, group=None):
    """The single collective of the step: allreduce(min) of the global ToI
    (a 1-element float64 tensor, CUDA under NCCL or CPU under gloo)."""
    import torch.distributed as dist
    if toi_tensor.is_cuda and host_staged(group):
        t = toi_tensor.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        toi_tensor.copy_(t)
        return toi_tensor
    dist.all_reduce(toi_tensor, op=dist.ReduceOp.MIN, group=group)
    return toi_tensor


def all_gather_counts(n: int, world: int, device, group=None):
    """all_gather of one int64 per rank (the candidate counts)."""
    import torch
    import torch.distributed as dist
    if host_staged(group):
        out = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(out, torch.tensor([n], dtype=torch.int64), group=group)
        return [int(x.item()) for x in out]
    cnt = torch.tensor([n], dtype=torch.int64, device=device)
    gathered = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(gathered, cnt, group=group)
    return [int(c) for c in gathered.cpu().tolist()]  # one read-back for all N counts


def bind_to_torch_stream(resident):
    """Stream contract of the multi-GPU layer: the context runs on torch's
    current stream of its device, so the context's kernels and copies
    (ccdk_copy_last_toi, ccdk_copy_keys_device, the narrow phase's sort of
    the received keys) are stream-ordered with the collectives torch issues
    (NCCL waits on the current stream; its outputs are ready for the next
    work enqueued there).  Without it, a context on its own non-blocking
    stream could allreduce a ToI before the copy lands, or sort keys
    all_to_all has not delivered yet."""
    import torch
    dev = torch.device(f"cuda:{resident.ctx.device}")
    handle = torch.cuda.current_stream(dev).cuda_stream
    # torch's default stream has handle 0, which ccdk_ctx_set_stream reads as
    # "a private stream of your own" — the very unordered case this contract
    # rules out; name it as the legacy default stream instead
    resident.ctx.set_stream(handle or CUDA_STREAM_LEGACY)
    return dev


class ShardedCcd:
    """Runs the device-resident CCD step for this rank's shard and combines
    the global ToI across ranks on the device."""

    def __init__(self, resident, rank: int, world: int):
        import torch
        self.resident = resident
        self.rank = rank
        self.world = world
        dev = bind_to_torch_stream(resident)
        self.toi = torch.full((1,), float("inf"), dtype=torch.float64, device=dev)

    def step(self, cfg):
        rep = self.resident.step(cfg, self.rank, self.world)
        if self.world > 1:
            self.resident.copy_toi_to(self.toi.data_ptr())
            allreduce_min_toi(self.toi)
        return rep

    def global_toi(self, rep) -> float:
        return float(self.toi.item()) if self.world > 1 else rep.toi.toi


def balanced_ranges(counts, world: int):
    """Rank r's slice [lo_r, hi_r) of the rank-ordered concatenation of all
    ranks' candidates (equal counts up to one)."""
    total = int(sum(int(c) for c in counts))
    return [(total * r // world, total * (r + 1) // world) for r in range(world)]


def exchange_splits(counts, rank: int, world: int):
    """all_to_all split sizes that move this rank's candidates (global range
    [off_rank, off_rank + counts[rank])) to the balanced owners."""
    counts = [int(c) for c in counts]
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    rng = balanced_ranges(counts, world)

    def overlap(a0, a1, b0, b1):
        return max(0, min(a1, b1) - max(a0, b0))

    send = [int(overlap(offs[rank], offs[rank + 1], lo, hi)) for lo, hi in rng]
    lo, hi = rng[rank]
    recv = [int(overlap(offs[s], offs[s + 1], lo, hi)) for s in range(world)]
    return send, recv


def _residue_count(n: int, first: int, world: int) -> int:
    """#{j in [0, n) : j = first (mod world)} for 0 <= first < world."""
    return 0 if first >= n else (n - 1 - first) // world + 1


def interleave_splits(counts, rank: int, world: int):
    """all_to_all split sizes of the interleaved policy: the candidate with
    global index g (rank-ordered concatenation) goes to rank g mod world."""
    counts = [int(c) for c in counts]
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    off, n = int(offs[rank]), counts[rank]
    send = [_residue_count(n, (d - off) % world, world) for d in range(world)]
    recv = [_residue_count(counts[s], (rank - int(offs[s])) % world, world) for s in range(world)]
    return send, recv


def rebalance_keys(keys, counts, rank: int, world: int, group=None, policy: str = "interleave"):
    """Move pair keys (a 1-D int64 tensor holding this rank's counts[rank]
    keys, any device) to their narrow-phase owners with one all_to_all_single
    (NCCL on GPUs, gloo on CPU).

    policy "interleave" (default): global candidate g goes to rank g mod N.
    Narrow-phase cost per query is heavy-tailed and spatially clustered (deep
    BFS trees next to the contact front), and the canonical order keeps
    neighbours together, so equal contiguous slices of it are NOT equal work:
    measured on C4 at N = 8 (profiles/r02_predict_scaling_C4.json) the
    heaviest contiguous slice took 4.5 ms of narrow phase against 0.34 ms for
    the lightest.  Striding spreads every cluster over all ranks.
    policy "contiguous": rank r takes the r-th equal slice."""
    import torch
    import torch.distributed as dist
    n = int(counts[rank])
    if policy == "interleave":
        send, recv = interleave_splits(counts, rank, world)
        off = int(sum(int(c) for c in counts[:rank]))
        # keys bound for rank d are j = (d - off) mod N, + N, + 2N, ... : one gather
        perm = torch.cat([torch.arange((d - off) % world, n, world, device=keys.device) for d in range(world)])
        keys = keys[:n][perm] if n else keys[:0]
    else:
        send, recv = exchange_splits(counts, rank, world)
    if keys.is_cuda and host_staged(group):
        out = torch.empty(sum(recv), dtype=keys.dtype)
        dist.all_to_all_single(out, keys[:sum(send)].cpu().contiguous(), output_split_sizes=recv,
                               input_split_sizes=send, group=group)
        return out.to(keys.device)
    out = torch.empty(sum(recv), dtype=keys.dtype, device=keys.device)
    dist.all_to_all_single(out, keys[:sum(send)].contiguous(), output_split_sizes=recv,
                           input_split_sizes=send, group=group)
    return out


class RebalancedCcd:
    """The multi-GPU CCD step with the narrow phase balanced by candidate
    count: sweep shard -> all_gather(counts) -> all_to_all(keys) -> classify +
    narrow on the balanced slice -> allreduce(min) of the ToI."""

    def __init__(self, resident, rank: int, world: int, group=None, policy: str = "interleave"):
        import torch
        self.resident = resident
        self.rank = rank
        self.world = world
        self.group = group
        self.policy = policy
        self.dev = bind_to_torch_stream(resident)
        self.toi = torch.full((1,), float("inf"), dtype=torch.float64, device=self.dev)
        self.keys = torch.empty(0, dtype=torch.int64, device=self.dev)

    def step(self, cfg):
        import torch
        import torch.distributed as dist
        n, nb, broad_ms = self.resident.broad(cfg, self.rank, self.world)
        counts = all_gather_counts(n, self.world, self.dev, self.group)
        if self.keys.numel() < max(n, 1):
            self.keys = torch.empty(max(n, 1), dtype=torch.int64, device=self.dev)
        self.resident.copy_keys(self.keys.data_ptr())
        mine = rebalance_keys(self.keys, counts, self.rank, self.world, self.group, self.policy)
        rep = self.resident.narrow_keys(cfg, mine.data_ptr(), mine.numel(), nb)
        self.resident.copy_toi_to(self.toi.data_ptr())
        allreduce_min_toi(self.toi, self.group)
        rep.shard_counts = counts
        rep.device["ms_broad"] = broad_ms  # box build + sweep shard + pair sort
        return rep

    def global_toi(self, rep) -> float:
        return float(self.toi.item())
