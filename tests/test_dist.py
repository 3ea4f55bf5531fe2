"""Multi-process (gloo, CPU) tests of the sharded paths: the halo plan and
exchange of the row-partitioned spmv, and batch sharding.  The per-rank
compute is a numpy stand-in for the libjv kernels (the CUDA product path is
exercised by the GPU tests); the products are compared bitwise with the
pinned oracle's single-process spmv."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1812_06160_b200 import dist as jd
from paper_1812_06160_b200 import workloads as W


class NumpyOps:
    """CPU stand-in for DeviceOps (same calls, torch CPU tensors)."""

    def tensor_i32(self, a):
        return torch.from_numpy(np.asarray(a, dtype=np.int64))

    def tensor_f64(self, a):
        return torch.from_numpy(np.asarray(a, dtype=np.float64).copy())

    def empty_f64(self, n):
        return torch.full((max(int(n), 1),), np.nan, dtype=torch.float64)

    def csr(self, rs, col, val):
        return (rs, col, val)

    def gather(self, idx, n, src, dst):
        dst[:n] = src[idx[:n]]

    def spmv_rows(self, csr, x, y, row_map):
        rs, col, val = csr
        out = oracle.spmv(rs, col, val, x.numpy()) if rs.size > 1 else np.zeros(0)
        y[row_map] = torch.from_numpy(out)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _spmv_worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = _matrix(name)
        bounds = jd.row_partition(a.row_start, world)
        plan = jd.plan_halo(a.row_start, a.col, a.val, bounds, rank, world)
        sp = jd.DistSpmv(plan, NumpyOps())
        x = np.random.default_rng(5).uniform(-1, 1, a.n)
        y = torch.zeros(plan.n_local, dtype=torch.float64)
        for rep in range(3):       # repeated products reuse the buffers
            sp.x_local.copy_(torch.from_numpy(x[plan.lo:plan.hi] * (rep + 1)))
            sp(sp.x_local, y)
        q.put((rank, plan.lo, plan.hi, y.numpy().copy(), plan.stats))
    except Exception as e:   # surface worker failures in the parent
        q.put((rank, "error", repr(e), None, None))
    finally:
        dist.destroy_process_group()


def _matrix(name):
    if name == "laplace7":
        return W.laplace7(9)
    if name == "rmat":
        return W.rmat(10, 2)
    if name == "random":
        return W.random_diag_dominant(700, row_nnz=9, seed=4)
    raise KeyError(name)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["laplace7", "rmat", "random"])
def test_dist_spmv_matches_serial(name, world):
    a = _matrix(name)
    x = np.random.default_rng(5).uniform(-1, 1, a.n) * 3
    want = oracle.spmv(a.row_start, a.col, a.val, x)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_spmv_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    y = np.full(a.n, np.nan)
    for rank, lo, hi, part, stats in got:
        assert lo != "error", hi
        y[lo:hi] = part
    assert np.array_equal(y, want)


def test_row_partition_balances_nnz():
    a = W.rmat(11, 1)
    for parts in (1, 2, 3, 8):
        b = jd.row_partition(a.row_start, parts)
        assert b[0] == 0 and b[-1] == a.n and np.all(np.diff(b) >= 0)
        nnz = np.diff(a.row_start[b])
        assert nnz.max() <= a.nnz / parts + np.diff(a.row_start).max()


def test_plan_layout_keeps_column_order():
    """Single-process plan pieces: ext indices are monotone per row and the
    ghost counts are what the rows read."""
    a = W.laplace7(6)
    bounds = jd.row_partition(a.row_start, 3)
    # rank 1 alone: emulate the peers' needs with the planner of each rank
    rs = np.asarray(a.row_start)
    for rank in range(3):
        lo, hi = bounds[rank], bounds[rank + 1]
        cols = a.col[rs[lo]:rs[hi]]
        owner = np.searchsorted(bounds, cols, side="right") - 1
        assert set(np.unique(owner)) <= {rank - 1, rank, rank + 1}


def test_shard_range_covers_batch():
    for world in (1, 2, 3, 4, 8):
        got = [list(jd.shard_range(64, r, world)) for r in range(world)]
        assert sum(got, []) == list(range(64))
        assert max(map(len, got)) - min(map(len, got)) <= 1


def test_plan_halo_all_matches_exchange():
    """In-process plans: what each rank sends is exactly what its peers
    receive, in the receivers' ghost order."""
    a = W.rmat(9, 3)
    plans = jd.plan_halo_all(a.row_start, a.col, 3, a.val)
    for p in plans:
        for q, off, m in p.recv:
            sent = dict((pp, idx) for pp, idx in plans[q].send)[p.rank]
            assert sent.size == m
            ghosts = sent + plans[q].lo
            # the receiver's ext slots [off, off+m) are the global columns `ghosts`
            lcol = a.col[a.row_start[p.lo]:a.row_start[p.hi]]
            used = np.unique(lcol[(lcol >= plans[q].lo) & (lcol < plans[q].hi)])
            assert np.array_equal(used, ghosts)


def _blockdiag_worker(rank, world, port, q):
    """Every rank owns exactly one diagonal block: no halo peers at all."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = W.block_diagonal([W.laplace7(5) for _ in range(world)])
        bounds = jd.row_partition(a.row_start, world)
        plan = jd.plan_halo(a.row_start, a.col, a.val, bounds, rank, world)
        sp = jd.DistSpmv(plan, NumpyOps())
        x = np.random.default_rng(1).uniform(-1, 1, a.n)
        y = torch.zeros(plan.n_local, dtype=torch.float64)
        sp.x_local.copy_(torch.from_numpy(x[plan.lo:plan.hi]))
        sp(sp.x_local, y)
        q.put((rank, plan.lo, plan.hi, y.numpy().copy(), plan.stats))
    except Exception as e:
        q.put((rank, "error", repr(e), None, None))
    finally:
        dist.destroy_process_group()


def test_dist_spmv_rank_without_peers():
    """A partition where ranks have no halo peers: the plan-time collective
    keeps every rank in the communicator, the product is still bitwise."""
    world = 3
    a = W.block_diagonal([W.laplace7(5) for _ in range(world)])
    x = np.random.default_rng(1).uniform(-1, 1, a.n)
    want = oracle.spmv(a.row_start, a.col, a.val, x)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_blockdiag_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    y = np.full(a.n, np.nan)
    for rank, lo, hi, part, stats in got:
        assert lo != "error", hi
        assert stats["peers"] == 0
        y[lo:hi] = part
    assert np.array_equal(y, want)


def _factor_records(shard, a):
    """Oracle stand-in for the device plan: level-ordered front end, serial
    factor and solves of the shard's block-diagonal matrix; per-system
    records cut out by BatchShard."""
    import hashlib
    fe = oracle.front_end(a.n, a.row_start, a.col, a.val)
    fval, bad = oracle.factor_serial(fe["row_start"], fe["col"], fe["val"], fe["diag"])
    assert bad == -1
    b = np.concatenate([np.random.default_rng(0).uniform(-1, 1, m) for m in shard.sizes])
    b = b[fe["perm"]]
    y = oracle.solve_forward(fe["row_start"], fe["col"], fval, b)
    x, _ = oracle.solve_backward(fe["row_start"], fe["col"], fval, fe["diag"], y)
    rows = shard.system_rows(fe["perm"])
    h = lambda v: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()
    return {sd: (h(shard.take_rows(fe["row_start"], fval, r)), h(x[r])) for sd, r in rows.items()}


def _batch_worker(rank, world, port, count, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = jd.BatchShard(count, rank, world)
        a = shard.assemble(lambda sd: W.rmat(9, sd))
        recs = shard.gather(_factor_records(shard, a))
        q.put((rank, shard.seeds, recs))
    except Exception as e:
        q.put((rank, "error", repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_batch_sharding_matches_single_process(world):
    """c5-style batch sharding over gloo ranks: every rank factors and solves
    its contiguous block of systems as one block-diagonal matrix; the
    gathered per-system factor / solution digests equal those of each system
    factored alone (and of the whole batch on one process)."""
    count = 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, count, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    owned = []
    for rank, seeds, recs in got:
        assert seeds != "error", recs
        owned += seeds
        assert sorted(recs) == list(range(count))
    assert sorted(owned) == list(range(count))
    one = jd.BatchShard(count)
    whole = _factor_records(one, one.assemble(lambda sd: W.rmat(9, sd)))
    for sd in range(count):
        alone = jd.BatchShard(1, first=sd)
        rec = _factor_records(alone, alone.assemble(lambda s: W.rmat(9, s)))[sd]
        assert whole[sd] == rec
        for _, _, recs in got:
            assert recs[sd] == rec
