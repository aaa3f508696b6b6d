"""ZeRO-3 partition + bucketed collectives: host-side logic on gloo, world 2."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2410_21316_b200 as D
from paper_2410_21316_b200.distributed import BucketedCollectives, ShardLayout, finalising_actions


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_layout_pads_ragged_last_rank():
    lay = ShardLayout.build(1000, 3, 128)
    assert lay.per_rank == 334 and lay.padded_total == 1002 and lay.num_buckets == 3
    assert lay.bucket_span(2) == (256, 78)
    assert lay.rank_of_bucket_piece(2, 2) == (76, 2)
    assert lay.rank_of_bucket_piece(0, 2) == (78, 0)
    lay = ShardLayout.build(70 * 10**9, 8, 10**8)
    assert lay.num_buckets == 88 and lay.bucket_span(87) == (8_700_000_000, 50_000_000)


def test_finalising_actions_cover_every_subgroup():
    for stride in (1, 2, 3, D.ALL_CPU):
        plan = D.build_plan(12, stride, static_ratio=0.25)
        fin = finalising_actions(plan)
        assert sorted(fin) == list(range(12))
        for sg, aid in fin.items():
            assert plan.actions[aid].lane.value != "cpu_compute"


def _rank_grads(rank: int, n: int) -> torch.Tensor:
    """Rank-specific bf16 grads whose sum's rounding depends on the order of
    the adds: ranks 0 and 2 hold +-x * 2^30 (they cancel), ranks 1 and 3
    small values that an earlier huge partial sum absorbs."""
    g = torch.Generator().manual_seed(7)
    big = torch.randn(n, generator=g) * 2.0 ** 30
    g = torch.Generator().manual_seed(1000 + rank)
    small = torch.randn(n, generator=g)
    x = {0: big, 2: -big}.get(rank % 4, small)
    return x.to(torch.bfloat16)


def _worker(rank, world, port, total, sg, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import optistate_oracle as O

        lay = ShardLayout.build(total, world, sg)
        coll = BucketedCollectives(lay)
        full = _rank_grads(rank, lay.padded_total)
        ok_rs = True
        for scale in (None, 1.0 / world):
            mine = torch.zeros(lay.per_rank, dtype=torch.bfloat16)
            coll.reduce_scatter_all(full, mine, scale=scale)
            lo = rank * lay.per_rank
            srcs = [_rank_grads(r, lay.padded_total)[lo:lo + lay.per_rank].view(torch.int16).numpy().view(np.uint16)
                    for r in range(world)]
            want = O.reduce_scatter(srcs, "bf16", 1.0 if scale is None else scale)
            ok_rs &= mine.view(torch.int16).numpy().view(np.uint16).tobytes() == want.tobytes()
        # all-gather: each rank contributes rank-tagged params
        shard_params = torch.full((lay.per_rank,), float(rank))
        gathered = torch.full((lay.padded_total,), -1.0)
        coll.all_gather_all(gathered, shard_params)
        want_g = torch.cat([torch.full((lay.per_rank,), float(r)) for r in range(world)])
        q.put((rank, ok_rs, torch.equal(gathered, want_g)))
    except Exception as e:  # report instead of hanging the parent
        import traceback

        q.put((rank, traceback.format_exc(), False))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total,sg,world", [(1000, 128, 2), (4096, 512, 2), (5000, 700, 4)])
def test_bucketed_collectives_gloo(total, sg, world):
    """Bucketed reduce-scatter = oracle.reduce_scatter (rank-order fp32 sum,
    one rounding, then the scale) bit for bit, at world 2 and 4; all-gather
    exact."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, sg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok_rs is True and ok_ag for _, ok_rs, ok_ag in res), res


def test_rank_order_reduce_differs_from_other_orders():
    """The fixture really exercises the order: summing the same four ranks'
    grads in another order changes some roundings."""
    from oracle import optistate_oracle as O

    srcs = [_rank_grads(r, 4096).view(torch.int16).numpy().view(np.uint16) for r in range(4)]
    a = O.reduce_scatter(srcs, "bf16")
    b = O.reduce_scatter(srcs[::-1], "bf16")
    assert a.tobytes() != b.tobytes()


def _step_worker(rank, world, port, q):
    """Per-rank host update of its shard equals the slice of a single-rank run."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import optistate_oracle as O

        total, sg = 10_000, 1_000
        full = O.initialize(total, sg, seed=3, lowp="bf16")
        lay = ShardLayout.build(total, world, sg)
        lo = rank * lay.per_rank
        n = sum(g.size for g in lay.ranks[rank])
        opt = D.ShardedOptimizer.allocate(n, sg, lowp="bf16")
        for name, key in (("_p", "p"), ("_m", "m"), ("_v", "v"), ("_g", "g"), ("_w", "w")):
            getattr(opt, name)[:] = full[key][lo:lo + n]
        D.sequential_oracle(opt, D.AdamHyper())
        w = torch.zeros(lay.per_rank, dtype=torch.int16)
        w[:n] = torch.from_numpy(opt.model16.view(np.int16))
        gathered = torch.zeros(lay.padded_total, dtype=torch.int16)
        BucketedCollectives(lay).all_gather_all(gathered.view(torch.bfloat16), w.view(torch.bfloat16))
        O.sequential_oracle(full)
        q.put((rank, gathered[:total].numpy().view(np.uint16).tobytes() == full["w"].tobytes()))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_sharded_update_then_gather_equals_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_step_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_plan_core_binding():
    from paper_2410_21316_b200.distributed import _parse_cpulist, plan_core_binding

    assert _parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    allowed = range(32)
    nodes = {0: list(range(16)), 1: list(range(16, 32))}
    # 8 GPUs, 4 per socket: each rank gets 4 cores of its own socket, disjoint
    gpu_nodes = [0, 0, 0, 0, 1, 1, 1, 1]
    got = [plan_core_binding(allowed, gpu_nodes, nodes, r) for r in range(8)]
    assert got[0] == [0, 1, 2, 3] and got[5] == [20, 21, 22, 23]
    assert sorted(c for g in got for c in g) == list(range(32))
    # no NUMA information: an even split of the allowed set
    got = [plan_core_binding(range(16), [-1] * 4, {}, r) for r in range(4)]
    assert got == [[0, 1, 2, 3], [4, 5, 6, 7], [8, 9, 10, 11], [12, 13, 14, 15]]
    # fewer cores than ranks, and a single rank keeps everything
    assert plan_core_binding([0, 1], [-1] * 4, {}, 3) == [1]
    assert plan_core_binding(range(8), [0], nodes, 0) == list(range(8))
    # a single rank on a two-socket host keeps its GPU's socket; unknown node: everything
    assert plan_core_binding(allowed, [1], nodes, 0) == list(range(16, 32))
    assert plan_core_binding(allowed, [-1], nodes, 0) == list(range(32))
    # a node whose CPUs are outside the allowed mask falls back to the mask
    assert plan_core_binding(range(4), [2, 2], {2: [40, 41]}, 1) == [2, 3]
