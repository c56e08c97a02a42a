"""Multi-GPU partitioning over free blocks of C.

Free (I/J) blocks of C are independent: partitioning is a sub-range of the scatter vectors
 and the K loop is never split, so ranks never reduce. The only
exchange is the initial distribution of A and B from the rank that holds them (torch.distributed
over NCCL/NVLink). Each rank then contracts into its own C shard through the same C-ABI call as
one GPU.

Distribution (`distribute`, the default of `contract_sharded` and bench.py): every operand is
cut into the distinct slabs the ranks' blocks read -- the operand narrowed to a rank's ranges of
the shard labels it carries -- and each slab goes to the group of ranks that read it:
  * the source sends it once, point to point, to the group's leader (unless the source is in
    the group itself), and
  * the leader broadcasts it within the group (an NCCL sub-communicator, `new_group`).
The source thus sends every byte of A and B at most once (its egress <= |A| + |B|, the same as
one ring broadcast of the full operands; less when its own slabs are read by nobody else), and a
rank receives only its own slabs (cfg5 at 8 GPUs: 1/4 of A and 1/2 of B, 6.1 GB instead of the
18.3 GB a full broadcast delivers to every rank). `broadcast_operands` keeps the full-broadcast
alternative. Slabs travel as dense tensors in the source operand's memory order, which the
source broadcasts first, so sender and receivers always agree on the layout.
"""
from __future__ import annotations

import math
from typing import Callable, Dict, List, Optional, Sequence, Tuple


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
    """Full-broadcast alternative: broadcast A and B (their flat storage) from `src`."""
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


def order_slowest_first(t) -> List[int]:
    """Dims of t ordered by decreasing stride (its memory order, outermost first)."""
    return sorted(range(t.dim()), key=lambda d: -abs(t.stride(d)))


# ---------------------------------------------------------------------------------------------
# slab distribution
# ---------------------------------------------------------------------------------------------

def slab_groups(world: int, lens: Dict[str, int], shard_labels: str, labels: str):
    """Distinct slabs of an operand with `labels`: [(ranges of the shard labels it carries,
    sorted ranks whose block reads that slab)], in a fixed order (every rank computes the same
    list)."""
    groups: Dict[tuple, List[int]] = {}
    for r in range(world):
        rg = shard_ranges(world, r, lens, shard_labels)
        key = tuple((x, rg[x]) for x in shard_labels if x in labels)
        groups.setdefault(key, []).append(r)
    return [(dict(k), sorted(v)) for k, v in sorted(groups.items())]


def plan_traffic(world: int, lens: Dict[str, int], shard_labels: str, operands, src: int = 0):
    """Modelled bytes of `distribute` for operands [(labels, element size)]: what the source
    sends (point-to-point sends plus one copy per broadcast it roots) and what each rank
    receives. A ring or tree broadcast sends each byte out of its root once."""
    out = {"src_egress": 0, "recv": [0] * world}
    for labels, esz in operands:
        for rg, ranks in slab_groups(world, lens, shard_labels, labels):
            nbytes = esz * math.prod(shard_shape(labels, lens, rg))
            if src not in ranks:
                out["src_egress"] += nbytes                  # send to the group's leader
            elif len(ranks) > 1:
                out["src_egress"] += nbytes                  # the source roots the broadcast
            for r in ranks:
                if r != src:
                    out["recv"][r] += nbytes
    return out


_groups: Dict[tuple, object] = {}


def _subgroup(ranks: Sequence[int]):
    """NCCL/gloo sub-communicator over `ranks` (created once; dist.new_group is collective over
    the default group, so every rank creates the same groups in the same order)."""
    import torch.distributed as dist
    key = tuple(ranks)
    if len(ranks) == dist.get_world_size():
        return None
    g = _groups.get(key)
    if g is None:
        g = _groups[key] = dist.new_group(list(ranks))
    return g


def _dense(view, order):
    """A dense copy of `view` laid out in memory order `order` (dims outermost first), and the
    view of that copy in the original dim order."""
    inv = sorted(range(len(order)), key=lambda i: order[i])
    base = view.permute(*order).contiguous()
    return base, base.permute(*inv)


def _empty(shape, order, dtype, device):
    import torch
    inv = sorted(range(len(order)), key=lambda i: order[i])
    base = torch.empty([shape[d] for d in order], dtype=dtype, device=device)
    return base, base.permute(*inv)


def distribute(labels_list: Sequence[str], tensors: Sequence, lens: Dict[str, int],
               shard_labels: str, world: int, rank: int, dtype=None, device=None, src: int = 0):
    """Give every rank the slabs of each operand that its block of C reads (module docstring).
    `tensors` are read on `src` only (None elsewhere). Returns ([slab of each operand, in its
    original dim order], elements this rank received, elements `src` sent)."""
    import torch.distributed as dist
    # the source's memory orders (and dtype), so both ends of every slab agree on its layout
    meta = [None]
    if rank == src:
        meta = [([order_slowest_first(t) for t in tensors], str(tensors[0].dtype).split(".")[-1])]
    dist.broadcast_object_list(meta, src)
    orders, dname = meta[0]
    if dtype is None:
        import torch
        dtype = getattr(torch, dname)
    # create every sub-communicator up front, in the same order on every rank
    plans = [slab_groups(world, lens, shard_labels, lab) for lab in labels_list]
    for plan in plans:
        for _, ranks in plan:
            if len(ranks) > 1:
                _subgroup(ranks)
    out, recv, sent = [], 0, 0
    for T, labels, order, plan in zip(tensors, labels_list, orders, plans):
        mine = None
        for rg, ranks in plan:
            inside = rank in ranks
            if rank != src and not inside:
                continue
            leader = src if src in ranks else ranks[0]
            shape = shard_shape(labels, lens, rg)
            if rank == src:
                base, view = _dense(narrow(T, labels, rg), order)
            else:
                base, view = _empty(shape, order, dtype, device)
            if src not in ranks:
                if rank == src:
                    dist.send(base, leader)
                    sent += base.numel()
                elif rank == leader:
                    dist.recv(base, src)
                    recv += base.numel()
            if len(ranks) > 1 and inside:
                dist.broadcast(base, leader, group=_subgroup(ranks))
                if rank == src:
                    sent += base.numel()
                elif rank != leader:
                    recv += base.numel()
            if inside:
                mine = view
        out.append(mine)
    return out, recv, sent


def distribute_slabs(spec: str, A, B, lens: Dict[str, int], shard_labels: str, world: int,
                     rank: int, dtype=None, device=None, src: int = 0):
    """A and B slabs for this rank (see `distribute`). Returns (A_slab, B_slab, elements
    received by this rank, elements sent by src)."""
    lc, la, lb = spec.split("-")
    (As, Bs), recv, sent = distribute([la, lb], [A, B], lens, shard_labels, world, rank,
                                      dtype, device, src)
    return As, Bs, recv, sent


def contract_sharded(spec: str, A, B, C=None, shard_labels: str = "abc", alpha: float = 1.0,
                     beta: float = 0.0, *, src: int = 0, gather: bool = False, device=None,
                     contract_fn: Optional[Callable] = None):
    """The process-group helper of SURVEY.md §8(b): C = alpha * A.B + beta * C over all ranks of
    the default process group, each rank computing the block of C given by its ranges of
    `shard_labels` (free labels of C).

    On rank `src`, A and B (and C when beta != 0 or gather=True) are the full tensors; on other
    ranks they may be None. The slabs each rank reads are distributed with `distribute`; when
    beta != 0 each rank also receives its block of C_old. Every rank returns its C block (dense,
    column-major over C's labels, on `device` -- default the current CUDA device). With
    gather=True the blocks are sent back and written into C on `src` (which then returns C).
    `contract_fn` defaults to the CUDA path (paper_1607_00291_b200.contract)."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    lc, la, lb = spec.split("-")
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    if contract_fn is None:
        import paper_1607_00291_b200 as tc
        contract_fn = tc.contract
    meta = [None]
    if rank == src:
        lens = {}
        for T, labels in ((A, la), (B, lb)):
            for x, n in zip(labels, T.shape):
                lens[x] = int(n)
        meta = [lens]
    dist.broadcast_object_list(meta, src)
    lens = meta[0]
    bad = [x for x in shard_labels if x not in lc]
    if bad:
        raise ValueError(f"shard labels {bad} are not free labels of C ({lc!r})")
    rg = shard_ranges(world, rank, lens, shard_labels)
    labels_list, tensors = [la, lb], [A, B]
    if beta != 0.0:
        labels_list.append(lc)
        tensors.append(C)
    slabs, _, _ = distribute(labels_list, tensors, lens, shard_labels, world, rank,
                             device=device, src=src)
    As, Bs = slabs[0], slabs[1]
    cshape = shard_shape(lc, lens, rg)
    colmajor = list(reversed(range(len(cshape))))
    base, Cs = _empty(cshape, colmajor, As.dtype, device)
    if beta != 0.0:
        Cs.copy_(slabs[2])
    contract_fn(spec, As, Bs, Cs, alpha, beta)
    if not gather:
        return Cs
    if rank == src:
        narrow(C, lc, rg).copy_(Cs)
        for r in range(world):
            if r == src:
                continue
            rr = shard_ranges(world, r, lens, shard_labels)
            b, v = _empty(shard_shape(lc, lens, rr), colmajor, As.dtype, device)
            dist.recv(b, r)
            narrow(C, lc, rr).copy_(v)
        return C
    dist.send(base, src)
    return Cs
