"""Multi-GPU partitioning over free blocks of C.

Free (I/J) blocks of C are independent: partitioning is a sub-range of the scatter vectors
 and the K loop is never split, so ranks never reduce. The only
exchange is the initial distribution of A and B from rank 0 (torch.distributed over NCCL/NVLink):
either a broadcast of the full operands (each rank then contracts zero-copy sub-views, base
pointer + narrowed lengths) or, with less volume, point-to-point slabs holding just what each
rank's block of C reads (distribute_slabs). Either way each rank contracts into its own C shard
through the same C ABI call as one GPU.
"""
from __future__ import annotations

import math
from typing import Callable, Dict, List, Sequence, Tuple


def shard_grid(world: int, shard_labels: str) -> Dict[str, int]:
    """Ways to split each shard label: 2 GPUs split the first label in 2, 4 split the first two,
    8 split all three (power-of-two worlds); other worlds split the first label `world` ways."""
    ways = {x: 1 for x in shard_labels}
    if world & (world - 1) == 0:
        w, i = world, 0
        while w > 1:
            ways[shard_labels[i % len(shard_labels)]] *= 2
            w //= 2
            i += 1
    else:
        ways[shard_labels[0]] = world
    return ways


def shard_ranges(world: int, rank: int, lens: Dict[str, int], shard_labels: str
                 ) -> Dict[str, Tuple[int, int]]:
    """[lo, hi) of every shard label for `rank` (row-major over shard_labels; balanced within
    one index when a length does not divide)."""
    ways = shard_grid(world, shard_labels)
    out, r = {}, rank
    for x in reversed(shard_labels):
        w = ways[x]
        q = r % w
        r //= w
        n = lens[x]
        out[x] = (q * n // w, (q + 1) * n // w)
    return out


def narrow(t, labels: str, ranges: Dict[str, Tuple[int, int]]):
    """Zero-copy sub-view of tensor t (labels) restricted to `ranges`."""
    for d, x in enumerate(labels):
        if x in ranges:
            lo, hi = ranges[x]
            t = t.narrow(d, lo, hi - lo)
    return t


def shard_shape(labels: str, lens: Dict[str, int], ranges) -> List[int]:
    return [(ranges[x][1] - ranges[x][0]) if x in ranges else lens[x] for x in labels]


def shard_flops(spec: str, lens: Dict[str, int], ranges) -> int:
    lc, la, lb = spec.split("-")
    n = 1
    for x in set(la) | set(lb) | set(lc):
        n *= (ranges[x][1] - ranges[x][0]) if x in ranges else lens[x]
    return 2 * n


def broadcast_operands(tensors: Sequence, src: int = 0) -> None:
    """The one exchange step: broadcast A and B (their flat storage) from `src`."""
    import torch.distributed as dist
    for t in tensors:
        dist.broadcast(t, src)


def contract_shard(spec: str, A, B, C_shard, ranges, alpha: float, beta: float,
                   contract_fn: Callable = None):
    """Contract this rank's block: A, B full operands (device), C_shard this rank's C block."""
    if contract_fn is None:
        import paper_1607_00291_b200 as tc
        contract_fn = tc.contract
    lc, la, lb = spec.split("-")
    return contract_fn(spec, narrow(A, la, ranges), narrow(B, lb, ranges), C_shard, alpha, beta)


def _order_slowest_first(t) -> List[int]:
    """Dims of t ordered by decreasing stride (its memory order, outermost first)."""
    return sorted(range(t.dim()), key=lambda d: -abs(t.stride(d)))


def distribute_slabs(spec: str, A, B, lens: Dict[str, int], shard_labels: str, world: int,
                     rank: int, dtype=None, device=None, order_a: Sequence[int] = None,
                     order_b: Sequence[int] = None, src: int = 0):
    """Lower-volume operand distribution: instead of broadcasting the full
    A and B, rank `src` sends every rank only the slabs its block of C reads -- A and B narrowed
    to that rank's ranges of the shard labels they carry -- each as one dense tensor
    over point-to-point send/recv. The slabs keep the operands' memory order (`order_a/b`: dims
    outermost first; default column-major, the workloads' layout). `src` keeps dense copies of
    its own slabs too, so every rank contracts the same layout. Returns (A_slab, B_slab,
    elements received by this rank). A and B are only read on `src` (None elsewhere)."""
    import torch
    import torch.distributed as dist
    lc, la, lb = spec.split("-")

    def order(T, given, labels):
        if given is not None:
            return list(given)
        if T is not None:
            return _order_slowest_first(T)
        return list(reversed(range(len(labels))))

    oa, ob = order(A, order_a, la), order(B, order_b, lb)

    def dense(view, o):
        inv = sorted(range(len(o)), key=lambda i: o[i])
        base = view.permute(*o).contiguous()
        return base, base.permute(*inv)

    def empty(labels, rg, o):
        shape = shard_shape(labels, lens, rg)
        base = torch.empty([shape[d] for d in o], dtype=dtype, device=device)
        inv = sorted(range(len(o)), key=lambda i: o[i])
        return base, base.permute(*inv)

    mine = shard_ranges(world, rank, lens, shard_labels)
    if rank == src:
        for r in range(world):
            if r == src:
                continue
            rg = shard_ranges(world, r, lens, shard_labels)
            for T, labels, o in ((A, la, oa), (B, lb, ob)):
                base, _ = dense(narrow(T, labels, rg), o)
                dist.send(base, r)
        _, a_mine = dense(narrow(A, la, mine), oa)
        _, b_mine = dense(narrow(B, lb, mine), ob)
        return a_mine, b_mine, 0
    abase, a_mine = empty(la, mine, oa)
    bbase, b_mine = empty(lb, mine, ob)
    dist.recv(abase, src)
    dist.recv(bbase, src)
    return a_mine, b_mine, abase.numel() + bbase.numel()
