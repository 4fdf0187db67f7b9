"""The N > 1 path on CPU: two gloo ranks run the slab-decomposed cycle
(oracle/distributed.py -- the algorithm of the r-slab CUDA path: ghost-plane
exchange, allgathered argmax + owner pair tests + allreduced PTL minimum,
plane-ordered PCG dots) and must reproduce the single-domain oracle: identical
cycle and stage counts and bitwise-equal fields for RKL2, identical PCG
iteration counts and fields to 1e-10 for BE; and BE+PCG is bitwise the same
for 1, 2, 3 and 8 slabs (GPU-count-invariant reductions).  Also pins the product's
host-side slab logic (geometry.slab_bounds / pack / flags) used by the CUDA
path."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

from helpers import oracle_aligned, oracle_scalar, oracle_geometry, soa
from oracle import ptl as optl
from paper_2403_01004_b200 import configs, geometry


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(name):
    if name == "c3":
        w = configs.c3(n=(11, 10, 16))
        op = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"])
        u = soa(w.fields["T"][..., None])
        return op, u, 300.0
    if name == "c2":
        w = configs.c2(n=(9, 8, 16))
        op = oracle_scalar(w.grid, w.bc, ncomp=3, vector_metric=True)
        return op, soa(w.fields["v"]), 200.0
    w = configs.c1(n=(9, 8, 16))
    op = oracle_scalar(w.grid, w.bc)
    return op, soa(w.fields["u"][..., None]), 60.0


def _worker(rank, world, port, name, kind, q):
    import torch.distributed as dist
    from oracle import distributed as od
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        op, u, ratio = _problem(name)
        slab = od.Slab(op.geom, rank, world)
        sop = od.SlabOperator(op, slab)
        dtE = sop.euler_dt()
        u_int = u[:, slab.i0:slab.i0 + slab.n].copy()
        out, rep = od.slab_cycle_operator(sop, kind, u_int, ratio * dtE, dtE, tol=1e-9)
        q.put((rank, slab.i0, out, [(r.dt, r.iters) for r in rep], dtE))
    finally:
        dist.destroy_process_group()


def _run(name, kind, world=2):
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, name, kind, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    return res


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_two_rank_rkl2_matches_single_domain(name):
    res = _run(name, "rkl2")
    op, u, ratio = _problem(name)
    dtE = op.euler_dt()
    assert all(r[4] == dtE for r in res), "allreduced Gershgorin bound differs"
    uo, repo = optl.cycle_operator(op, optl.OracleScheme("rkl2"), u, ratio * dtE, dt_euler=dtE)
    for _, i0, out, rep, _ in res:
        assert rep == [(r.dt, r.iters) for r in repo]
        assert np.array_equal(out, uo[:, i0:i0 + out.shape[1]])


def test_two_rank_be_pcg_matches_single_domain():
    res = _run("c3", "backward_euler")
    op, u, ratio = _problem("c3")
    dtE = op.euler_dt()
    uo, repo = optl.cycle_operator(op, optl.OracleScheme("backward_euler", tol=1e-9), u, ratio * dtE, dt_euler=dtE)
    for _, i0, out, rep, _ in res:
        assert [x[1] for x in rep] == [r.iters for r in repo]
        ref = uo[:, i0:i0 + out.shape[1]]
        assert np.linalg.norm(out - ref) <= 1e-10 * np.linalg.norm(ref)


def _worker_c4(rank, world, port, kind, q):
    import torch.distributed as dist
    from oracle import distributed as od
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        w = configs.c4(n=(16, 10, 16))
        op = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"])
        u = soa(w.fields["T"][..., None])
        slab = od.Slab(op.geom, rank, world)
        sop = od.SlabOperator(op, slab)
        dtE = sop.euler_dt()
        u_int = u[:, slab.i0:slab.i0 + slab.n].copy()
        out, rep = od.slab_cycle_operator(sop, kind, u_int, 1e3 * dtE, dtE, tol=1e-9)
        q.put((rank, slab.i0, out, [(r.dt, r.iters) for r in rep], dtE))
    finally:
        dist.destroy_process_group()


def test_be_pcg_bitwise_invariant_to_slab_count():
    """C4 recipe (BE + Jacobi PCG, PTL cycling): 1, 2, 3 and 8 slabs give the
    same iteration counts per cycle and bitwise the same field -- the PCG
    inner products are summed per plane and then over the global planes in
    order, whatever the split."""
    ctx = mp.get_context("fork")
    results = {}
    for world in (1, 2, 3, 8):
        q = ctx.Queue()
        port = _free_port()
        ps = [ctx.Process(target=_worker_c4, args=(r, world, port, "backward_euler", q)) for r in range(world)]
        for p in ps:
            p.start()
        res = sorted(q.get(timeout=300) for _ in range(world))
        for p in ps:
            p.join(timeout=60)
            assert p.exitcode == 0
        assert all(r[3] == res[0][3] for r in res)
        results[world] = (np.concatenate([r[2] for r in res], axis=1), res[0][3])
    f1, rep1 = results[1]
    assert sum(it for _, it in rep1) > 20
    for world in (2, 3, 8):
        f, rep = results[world]
        assert rep == rep1, world
        assert np.array_equal(f, f1), world


@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_product_slab_tables_are_global_rows(nranks):
    """geometry.pack for a slab == the global tables' rows (ghost rows included)."""
    w = configs.c3(n=(17, 6, 8))
    gt = geometry.global_tables(w.grid, w.bc)
    full = geometry.pack(gt)
    n0, n1 = gt.shape[0], gt.shape[1]
    A = (n0 + 2) * n1
    covered = 0
    for r in range(nranks):
        i0, n = geometry.slab_bounds(n0, nranks, r)
        covered += n
        lo, hi = r > 0, r < nranks - 1
        tab = geometry.pack(gt, i0, n, lo, hi)
        fl = geometry.flags(gt, i0, n, lo, hi)
        assert fl[11] == n0 and fl[12] == i0 and fl[9] == lo and fl[10] == hi
        a = (n + 2) * n1
        # first 2-D table (W0): rows i0-1 .. i0+n of the global table (ghosts only where a slab exists)
        glob = full[:A].reshape(n0 + 2, n1)
        loc = tab[:a].reshape(n + 2, n1)
        assert np.array_equal(loc[1:-1], glob[1 + i0:1 + i0 + n])
        if lo:
            assert np.array_equal(loc[0], glob[i0])
        if hi:
            assert np.array_equal(loc[-1], glob[i0 + n + 1])
    assert covered == n0
