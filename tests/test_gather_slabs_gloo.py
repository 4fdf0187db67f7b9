"""device.gather_slabs on two gloo CPU ranks: the slabs of a multi-rank
context (r-slabs along axis 0, phi-slabs along axis 2, ragged sizes) are
all-gathered back into the global array on every rank -- the path every
host-Field API call (cycle_operator, split_advance, to_field) ends in on N
GPUs (to_field must not reshape a slab as the global grid)."""
import multiprocessing as mp
import socket
import types

import numpy as np
import pytest


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, axis, q):
    import torch.distributed as dist
    from paper_2403_01004_b200 import device, geometry
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        shape = (7, 5, 11)
        glob = np.arange(np.prod(shape) * 3, dtype=float).reshape(shape + (3,))
        nax = shape[axis]
        k0, n = geometry.slab_bounds(nax, world, rank)
        dg = types.SimpleNamespace(ctx=types.SimpleNamespace(nranks=world, device=0), global_shape=shape,
                                   phi=(k0, n) if axis == 2 else None)
        local = glob[:, :, k0:k0 + n] if axis == 2 else glob[k0:k0 + n]
        out = device.gather_slabs(dg, np.ascontiguousarray(local))
        q.put((rank, bool(np.array_equal(out, glob))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("axis", [0, 2])
@pytest.mark.parametrize("world", [2, 3])
def test_gather_slabs(axis, world):
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, axis, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)
