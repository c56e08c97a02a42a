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


def _run_world(target, world, *extra):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + extra) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return q.get(timeout=10)


def _rowmajor(t):
    """t re-stored row-major (last dim fastest), same values and dim order."""
    return t.contiguous()


def _worker_slabs(rank, world, port, q, layout):
    """The slab distribution (dist.distribute_slabs: point-to-point to each slab group's leader,
    then a broadcast within the group): the shards must assemble to the single result; each rank
    receives exactly its slab volume; the source sends A and B at most once."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = W.cfg5(big=6, small=4)
        case.dist = "int"
        A = B = None
        if rank == 0:
            A, B, _ = W.make_tensors(case, "cpu")
            if layout == "rowmajor":   # the receivers must use the sender's layout
                A, B = _rowmajor(A), _rowmajor(B)
        As, Bs, got, sent = tdist.distribute_slabs(case.spec, A, B, case.lens, "abc", world,
                                                   rank, device="cpu")
        rg = tdist.shard_ranges(world, rank, case.lens, "abc")
        expect = (math.prod(tdist.shard_shape(case.lab_a, case.lens, rg)) +
                  math.prod(tdist.shard_shape(case.lab_b, case.lens, rg)))
        cshape = tdist.shard_shape(case.lab_c, case.lens, rg)
        C = W.colmajor_view(torch.full((math.prod(cshape),), float("nan"), dtype=torch.float64),
                            cshape)
        _oracle_contract(case.spec, As, Bs, C, case.alpha, case.beta)
        shards = [None] * world
        dist.all_gather_object(shards, (rg, C.contiguous().numpy(), got, expect, sent))
        if rank == 0:
            full = W.make_tensors(case, "cpu")
            ref = full[2].clone()
            _oracle_contract(case.spec, full[0], full[1], ref, case.alpha, case.beta)
            out = np.full(ref.shape, np.nan)
            ok = True
            model = tdist.plan_traffic(world, case.lens, "abc",
                                       [(case.lab_a, 1), (case.lab_b, 1)])
            for r, (g, c, n_got, n_exp, _) in enumerate(shards):
                out[g["a"][0]:g["a"][1], g["b"][0]:g["b"][1], g["c"][0]:g["c"][1]] = c
                ok &= n_got == (0 if r == 0 else n_exp)
                ok &= model["recv"][r] == (0 if r == 0 else n_exp)
                ok &= n_exp < full[0].numel() + full[1].numel()
            # the source sends every element of A and B at most once (one broadcast's egress)
            ok &= shards[0][4] == model["src_egress"] <= full[0].numel() + full[1].numel()
            q.put(bool(ok and np.array_equal(out, ref.numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("layout", ["colmajor", "rowmajor"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_gloo_slab_distribution_equals_single(world, layout):
    assert _run_world(_worker_slabs, world, layout) is True


def test_slab_traffic_model_cfg5():
    """cfg5 at full size: the source's egress and each rank's receive volume (bytes, fp64)."""
    case = W.cfg5()
    A = 8 * math.prod(case.shape(case.lab_a))
    B = 8 * math.prod(case.shape(case.lab_b))
    for world, egress, recv in ((2, A // 2 + B, A // 2 + B), (4, 3 * A // 4 + B, A // 4 + B),
                                (8, A + B, A // 4 + B // 2)):
        m = tdist.plan_traffic(world, case.lens, "abc", [(case.lab_a, 8), (case.lab_b, 8)])
        assert m["src_egress"] == egress <= A + B, world
        assert m["recv"][0] == 0 and all(r == recv for r in m["recv"][1:]), world


def _worker_sharded(rank, world, port, q, beta, gather):
    """tc.dist.contract_sharded with the oracle as the per-rank contraction:
    the operands exist on rank 0 only; beta != 0 ships each rank its block of C_old."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = W.cfg5(big=6, small=4)
        case.dist, case.beta, case.c_init = "int", beta, "dist" if beta else "nan"
        A = B = C = None
        if rank == 0:
            A, B, C = W.make_tensors(case, "cpu")
            C0 = C.clone()
        Cs = tdist.contract_sharded(case.spec, A, B, C, "abc", 2.0, beta, gather=gather,
                                    device="cpu", contract_fn=_oracle_contract)
        rg = tdist.shard_ranges(world, rank, case.lens, "abc")
        shards = [None] * world
        dist.all_gather_object(shards, (rg, tdist.narrow(Cs, case.lab_c, rg).contiguous().numpy()
                                        if (gather and rank == 0) else Cs.contiguous().numpy()))
        if rank == 0:
            ref = C0.clone()
            _oracle_contract(case.spec, A, B, ref, 2.0, beta)
            out = np.full(ref.shape, np.nan)
            for g, c in shards:
                out[g["a"][0]:g["a"][1], g["b"][0]:g["b"][1], g["c"][0]:g["c"][1]] = c
            ok = np.array_equal(out, ref.numpy())
            if gather:
                ok &= torch.equal(C, ref)
            q.put(bool(ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("beta,gather", [(0.0, False), (0.5, True)])
@pytest.mark.parametrize("world", [2, 8])
def test_gloo_contract_sharded(world, beta, gather):
    assert _run_world(_worker_sharded, world, beta, gather) is True
