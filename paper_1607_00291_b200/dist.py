"""Multi-GPU partitioning over free blocks of C.

Free (I/J) blocks of C are independent: partitioning is a sub-range of the scatter vectors
 and the K loop is never split, so ranks never reduce. The only
collective is the initial NCCL broadcast of A and B from rank 0 (torch.distributed, NVLink).
Each rank then contracts its shard with zero-copy sub-views of A and B (base pointer + narrowed
lengths) into its own C shard, through the same C ABI call as one GPU.
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
