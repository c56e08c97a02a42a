"""N>1 host logic on CPU: shard ranges cover C exactly once, and a world-size-2 gloo run of the
multi-GPU protocol (rank-0 operands -> broadcast -> per-rank shard contraction on zero-copy
views -> gather) reproduces the single-process result. The per-shard contraction here is the
oracle (test-side); on GPUs the same dist.contract_shard calls the CUDA path."""
import itertools
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W
from paper_1607_00291_b200 import dist as tdist


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_ranges_partition_free_blocks(world):
    lens = {"a": 48, "b": 48, "c": 48, "d": 48, "i": 24, "j": 24, "k": 24, "l": 24, "m": 24}
    seen = np.zeros((48, 48, 48), dtype=np.int32)
    total = 0
    for r in range(world):
        rg = tdist.shard_ranges(world, r, lens, "abc")
        seen[rg["a"][0]:rg["a"][1], rg["b"][0]:rg["b"][1], rg["c"][0]:rg["c"][1]] += 1
        total += tdist.shard_flops("abcijk-abdilm-dclmjk", lens, rg)
    assert (seen == 1).all()
    assert total == W.cfg5().flops()


def test_shard_grid_matches_survey_plan():
    assert tdist.shard_grid(2, "abc") == {"a": 2, "b": 1, "c": 1}
    assert tdist.shard_grid(4, "abc") == {"a": 2, "b": 2, "c": 1}
    assert tdist.shard_grid(8, "abc") == {"a": 2, "b": 2, "c": 2}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_contract(spec, A, B, C, alpha, beta):
    import oracle
    oracle.contract(spec, A, B, C, alpha, beta)
    return C


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = W.cfg5(big=6, small=4)
        shape_a, shape_b = case.shape(case.lab_a), case.shape(case.lab_b)
        if rank == 0:
            A, B, _ = W.make_tensors(case, "cpu")
        else:
            A = W.colmajor_view(torch.empty(math.prod(shape_a), dtype=torch.float64), shape_a)
            B = W.colmajor_view(torch.empty(math.prod(shape_b), dtype=torch.float64), shape_b)
        tdist.broadcast_operands([torch.as_strided(A, (A.numel(),), (1,)),
                                  torch.as_strided(B, (B.numel(),), (1,))], 0)
        rg = tdist.shard_ranges(world, rank, case.lens, "abc")
        cshape = tdist.shard_shape(case.lab_c, case.lens, rg)
        C = W.colmajor_view(torch.full((math.prod(cshape),), float("nan"), dtype=torch.float64),
                            cshape)
        tdist.contract_shard(case.spec, A, B, C, rg, case.alpha, case.beta,
                             contract_fn=_oracle_contract)
        shards = [None] * world
        dist.all_gather_object(shards, (rg, C.contiguous().numpy()))
        if rank == 0:
            full = W.make_tensors(case, "cpu")
            ref = full[2].clone()
            _oracle_contract(case.spec, full[0], full[1], ref, case.alpha, case.beta)
            out = np.full(ref.shape, np.nan)
            for r, c in shards:
                out[r["a"][0]:r["a"][1], r["b"][0]:r["b"][1], r["c"][0]:r["c"][1]] = c
            q.put(bool(np.array_equal(out, ref.numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_sharded_equals_single(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def _worker_slabs(rank, world, port, q):
    """Same protocol with the lower-volume distribution: rank 0 sends each rank only its A and
    B slabs (dist.distribute_slabs); the shards must still assemble to the single result, and
    each rank must have received exactly its slab volume."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = W.cfg5(big=6, small=4)
        A = B = None
        if rank == 0:
            A, B, _ = W.make_tensors(case, "cpu")
        As, Bs, got = tdist.distribute_slabs(case.spec, A, B, case.lens, "abc", world, rank,
                                             dtype=torch.float64, device="cpu")
        rg = tdist.shard_ranges(world, rank, case.lens, "abc")
        expect = (math.prod(tdist.shard_shape(case.lab_a, case.lens, rg)) +
                  math.prod(tdist.shard_shape(case.lab_b, case.lens, rg)))
        cshape = tdist.shard_shape(case.lab_c, case.lens, rg)
        C = W.colmajor_view(torch.full((math.prod(cshape),), float("nan"), dtype=torch.float64),
                            cshape)
        _oracle_contract(case.spec, As, Bs, C, case.alpha, case.beta)
        shards = [None] * world
        dist.all_gather_object(shards, (rg, C.contiguous().numpy(), got, expect))
        if rank == 0:
            full = W.make_tensors(case, "cpu")
            ref = full[2].clone()
            _oracle_contract(case.spec, full[0], full[1], ref, case.alpha, case.beta)
            out = np.full(ref.shape, np.nan)
            ok = True
            for r, (g, c, n_got, n_exp) in enumerate(shards):
                out[g["a"][0]:g["a"][1], g["b"][0]:g["b"][1], g["c"][0]:g["c"][1]] = c
                ok &= (n_got == (0 if r == 0 else n_exp))
                # less than the full operands whenever the rank's block is a proper sub-block
                ok &= n_exp < full[0].numel() + full[1].numel()
            q.put(bool(ok and np.array_equal(out, ref.numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_slab_distribution_equals_single(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_slabs, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True
