"""Device-side handles: context (one per GPU / rank), grids and fields.

Thin RAII wrappers over the C ABI.  A ``DeviceField`` lives in HBM in the
SoA layout of the library; ``upload``/``download`` convert from/to the
reference ``Field`` layout (component innermost).  With ``nranks > 1`` every
rank holds its axis-0 (r) slab (``geometry.slab_bounds``).
"""
from __future__ import annotations

import ctypes
import os
from ctypes import byref, c_double, c_int64, c_void_p

import numpy as np

from . import _lib, geometry, mesh


class Context:
    def __init__(self, device: int = 0, nranks: int = 1, rank: int = 0, nccl_uid: bytes | None = None,
                 detached: bool = False, axis: int = 0):
        """``detached``: test hook -- a slab rank with no communicator
        (collectives skipped; ghost planes / columns set with
        DeviceField.set_ghost / set_ghost_cols).  ``axis``: the slab
        decomposition, 0 = r-slabs, 2 = phi-slabs (BASELINE C4's split)."""
        L = _lib.lib()
        h = c_void_p()
        if detached:
            _lib.check(L.pc_ctx_create_detached(int(device), int(nranks), int(rank), byref(h)),
                       "pc_ctx_create_detached")
        else:
            uid = None
            if nccl_uid is not None:
                uid = ctypes.create_string_buffer(bytes(nccl_uid), 128)
            _lib.check(L.pc_ctx_create(int(device), int(nranks), int(rank), uid, byref(h)), "pc_ctx_create")
        self.handle = h
        self.device = device
        self.nranks = nranks
        self.rank = rank
        self.axis = int(axis)
        if self.axis != 0:
            _lib.check(L.pc_ctx_set_decomposition(h, self.axis), "pc_ctx_set_decomposition")
        self._grids = {}
        self._pinned = []

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            for a in self._pinned:
                _lib.lib().pc_host_unregister(a.ctypes.data)
            self._pinned = []
            self._grids = {}
            _lib.lib().pc_ctx_destroy(self.handle)
            self.handle = None

    def sync(self):
        _lib.check(_lib.lib().pc_ctx_sync(self.handle), "sync")

    def enable_timing(self, on: bool = True):
        _lib.lib().pc_ctx_enable_timing(self.handle, int(on))

    def mark(self, slot: int):
        """Record a CUDA event on the library stream (device timing)."""
        _lib.check(_lib.lib().pc_ctx_mark(self.handle, int(slot)), "mark")

    def elapsed_ms(self, a: int, b: int) -> float:
        v = c_double()
        _lib.check(_lib.lib().pc_ctx_elapsed(self.handle, int(a), int(b), byref(v)), "elapsed")
        return v.value

    def reset_stats(self):
        _lib.lib().pc_ctx_reset_stats(self.handle)

    def stats(self):
        ms = c_double()
        sl = c_int64()
        tot = c_int64()
        _lib.lib().pc_ctx_stats(self.handle, byref(ms), byref(sl), byref(tot))
        return {"stage_ms": ms.value, "stage_launches": sl.value, "launches": tot.value}

    # sts_f12 / sts_f12w: the fused stage-1+2 launch of the 7-point march
    # (without / with the u1 write); their cell-updates count both stages
    # (sts_af12 / sts_af12w: the same for the aligned TMA march)
    KINDS = ("sts_scalar", "sts_aligned", "pcg_scalar", "pcg_aligned", "sts_f12", "sts_f12w", "sts_af12",
             "sts_af12w")

    def stats_by_kind(self):
        """{kind: {ms, launches, cell_updates}} of the timed hot loops."""
        out = {}
        for q, name in enumerate(self.KINDS):
            ms, nl, cu = c_double(), c_int64(), c_int64()
            _lib.check(_lib.lib().pc_ctx_stats_kind(self.handle, q, byref(ms), byref(nl), byref(cu)), "stats")
            out[name] = {"ms": ms.value, "launches": nl.value, "cell_updates": cu.value}
        return out

    def pin(self, arr: np.ndarray):
        """Page-lock a host array (kept pinned for the context's lifetime);
        arrays already in page-locked memory (pinned_empty) are left alone."""
        if is_page_locked(arr):
            return arr
        _lib.check(_lib.lib().pc_host_register(arr.ctypes.data, arr.nbytes), "pin")
        self._pinned.append(arr)
        return arr

    def unpin(self, arr: np.ndarray):
        for q, a in enumerate(self._pinned):
            if a is arr:
                _lib.lib().pc_host_unregister(arr.ctypes.data)
                del self._pinned[q]
                return

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _lib.check(_lib.lib().pc_nccl_unique_id(buf), "ncclGetUniqueId")
        return buf.raw


_default: Context | None = None


def default_context() -> Context:
    global _default
    if _default is None or _default.handle is None:
        _default = Context(int(os.environ.get("PARACYCLE_DEVICE", "0")))
    return _default


def set_default_context(ctx: Context):
    global _default
    _default = ctx


class _PinnedBlock:
    """A page-locked host block; returned to the cache when the last numpy
    array (or view) over it is garbage-collected."""

    def __init__(self, cache, ptr, nbytes):
        self.cache, self.ptr, self.nbytes = cache, ptr, nbytes

    def __del__(self):
        try:
            self.cache._release(self)
        except Exception:
            pass


class _PinnedCache:
    """Caching allocator of page-locked host memory for downloads: a fresh
    pageable array costs a page fault per page on the device->host copy
    (~4 GB/s), a recycled pinned block copies at PCIe speed (~50 GB/s).
    Blocks are reused by exact size; at most ``limit`` bytes stay cached."""

    def __init__(self, limit=96 << 30):
        self.free = {}
        self.cached = 0
        self.limit = limit

    def empty(self, shape):
        n = int(np.prod(shape)) * 8
        lst = self.free.get(n)
        if lst:
            blk = lst.pop()
            self.cached -= n
        else:
            p = c_void_p()
            if not _lib.alive() or _lib.lib().pc_host_alloc(n, byref(p)) != 0 or not p.value:
                return np.empty(shape)  # no page-locked memory left: pageable fallback (host buffer only)
            blk = _PinnedBlock(self, p.value, n)
        buf = (ctypes.c_byte * n).from_address(blk.ptr)
        buf._block = blk  # keeps the block alive as long as any array over it
        return np.frombuffer(buf, dtype=np.float64).reshape(shape)

    def _release(self, blk):
        if not _lib.alive():
            return
        if self.cached + blk.nbytes <= self.limit:
            fresh = _PinnedBlock(self, blk.ptr, blk.nbytes)
            blk.ptr = None
            self.free.setdefault(fresh.nbytes, []).append(fresh)
            self.cached += fresh.nbytes
        elif blk.ptr:
            _lib.lib().pc_host_free(blk.ptr)
            blk.ptr = None


_pinned = _PinnedCache()


def is_page_locked(arr: np.ndarray) -> bool:
    """True if the array lives in a block of the pinned cache."""
    b = arr
    while b is not None:
        if getattr(b, "_block", None) is not None:
            return True
        b = getattr(b, "base", None)
    return False


def pinned_empty(shape) -> np.ndarray:
    """An uninitialised float64 array in (cached) page-locked host memory."""
    return _pinned.empty(tuple(int(x) for x in shape))


class DeviceGrid:
    """A grid (+ boundary condition) resident on one rank: metric tables and
    the slab geometry."""

    def __init__(self, grid, bc, ctx: Context | None = None, force_ghosts: bool = False):
        """``force_ghosts`` (test hook): a single rank reads its neighbours
        from ghost planes (r-slabs, periodic axis 0) or ghost columns
        (phi-slabs) filled by the (self) NCCL exchange instead of wrapping
        in-kernel."""
        ctx = ctx or default_context()
        self.ctx = ctx
        self.grid = grid
        self.bc = bc
        gt = geometry.global_tables(grid, bc)
        self.tables_global = gt
        n0 = gt.shape[0]
        P, r = ctx.nranks, ctx.rank
        if P > n0:
            raise ValueError(f"{P} ranks but only {n0} axis-0 planes")
        self.global_shape = gt.shape
        self.phi = None  # (k0, n) of a phi-slab rank
        if ctx.axis == 2 and (P > 1 or force_ghosts):
            n2 = gt.shape[2]
            if P > n2:
                raise ValueError(f"{P} ranks but only {n2} phi columns")
            self.phi = geometry.slab_bounds(n2, P, r)
            i0, n0l = 0, n0
            self.ghost_lo = self.ghost_hi = False
            self.i0, self.n0_local = i0, n0l
            self.shape = (n0, gt.shape[1], self.phi[1] + 2)  # + ghost columns
            self.host_shape = (n0, gt.shape[1], self.phi[1])
            tab = geometry.pack(gt, phi=self.phi)
            fl = geometry.flags(gt, phi=self.phi)
        else:
            i0, n0l = geometry.slab_bounds(n0, P, r)
            per0 = gt.periodic[0]
            self.ghost_lo = (P > 1 and (r > 0 or per0)) or (force_ghosts and per0)
            self.ghost_hi = (P > 1 and (r < P - 1 or per0)) or (force_ghosts and per0)
            self.i0, self.n0_local = i0, n0l
            self.shape = (n0l, gt.shape[1], gt.shape[2])
            self.host_shape = self.shape
            tab = geometry.pack(gt, i0, n0l, self.ghost_lo, self.ghost_hi)
            fl = geometry.flags(gt, i0, n0l, self.ghost_lo, self.ghost_hi)
        shp = (c_int64 * 3)(*self.shape)
        L = _lib.lib()
        if L.pc_grid_table_size(shp) != tab.size:
            raise RuntimeError("table layout mismatch between geometry.py and the library")
        h = c_void_p()
        _lib.check(L.pc_grid_create(ctx.handle, shp, fl.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                    _lib.dptr(tab), tab.size, byref(h)), "pc_grid_create")
        self.handle = h
        self.pinned = gt.pinned

    @property
    def ncells(self) -> int:
        """Cells this rank owns (phi-slabs: without the ghost columns)."""
        return int(np.prod(self.host_shape))

    def local_slice(self, values: np.ndarray) -> np.ndarray:
        """This rank's slab of a global grid-shaped array."""
        if self.phi is not None:
            k0, n = self.phi
            return values[:, :, k0:k0 + n]
        if self.ctx.nranks == 1:
            return values
        return values[self.i0:self.i0 + self.n0_local]

    def __del__(self):
        try:
            if _lib.alive() and self.handle is not None and self.ctx.handle is not None:
                _lib.lib().pc_grid_destroy(self.handle)
        except Exception:
            pass


def device_grid(grid, bc, ctx: Context | None = None) -> DeviceGrid:
    ctx = ctx or default_context()
    key = (id(grid), id(bc))
    hit = ctx._grids.get(key)
    if hit is not None and hit[0] is grid and hit[1] is bc:
        return hit[2]
    dg = DeviceGrid(grid, bc, ctx)
    ctx._grids[key] = (grid, bc, dg)
    return dg


def _embed3(values: np.ndarray, dims: int) -> np.ndarray:
    """(grid shape..., ncomp) -> (n0, n1, n2, ncomp) for 1-D/2-D grids."""
    v = values
    while v.ndim < 4:
        v = v[..., None, :] if dims < 3 else v
        dims += 1
    return v


def require_gather_group():
    """Host-Field results on more than one rank are gathered with
    torch.distributed: raise before any work when no process group exists."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        raise ValueError("host Fields on a multi-rank context need an initialised torch.distributed process group "
                         "(the slabs are gathered back to a global Field); pass DeviceFields instead")


def gather_slabs(dgrid: DeviceGrid, local: np.ndarray) -> np.ndarray:
    """All-gather the axis-0 slabs (n0_local, n1, n2, ncomp) of every rank
    into the global (n0, n1, n2, ncomp) array (geometry.slab_bounds order)."""
    import torch
    import torch.distributed as dist
    require_gather_group()
    P = dgrid.ctx.nranks
    ax = 2 if dgrid.phi is not None else 0
    nax = dgrid.global_shape[ax]
    bounds = [geometry.slab_bounds(nax, P, r) for r in range(P)]
    nmax = max(n for _, n in bounds)
    loc = np.moveaxis(np.asarray(local), ax, 0)
    tail = loc.shape[1:]
    dev = torch.device("cuda", dgrid.ctx.device) if dist.get_backend() == "nccl" else torch.device("cpu")
    buf = torch.zeros((nmax,) + tuple(tail), dtype=torch.float64, device=dev)
    buf[:loc.shape[0]] = torch.from_numpy(np.ascontiguousarray(loc)).to(dev)
    parts = [torch.empty_like(buf) for _ in range(P)]
    dist.all_gather(parts, buf)
    out = np.empty((nax,) + tuple(tail))
    for (i0, n), p in zip(bounds, parts):
        out[i0:i0 + n] = p[:n].cpu().numpy()
    return np.ascontiguousarray(np.moveaxis(out, 0, ax))


class DeviceField:
    def __init__(self, dgrid: DeviceGrid, ncomp: int = 1):
        self.dgrid = dgrid
        self.ncomp = int(ncomp)
        h = c_void_p()
        _lib.check(_lib.lib().pc_field_create(dgrid.handle, self.ncomp, byref(h)), "pc_field_create")
        self.handle = h
        self._holds = []  # host arrays of in-flight asynchronous copies (released by wait())

    @property
    def shape(self):
        return self.dgrid.shape

    def _host_shape(self, layout):
        hs = tuple(self.dgrid.host_shape)
        return hs + (self.ncomp,) if layout == _lib.LAYOUT_AOS else (self.ncomp,) + hs

    def upload(self, values: np.ndarray, layout: int = _lib.LAYOUT_AOS, async_: bool = False):
        """values: local slab, (n0, n1, n2, ncomp) AoS (or (ncomp, n0, n1, n2) SoA).
        ``async_``: the copy runs on the context's copy stream and the field's
        next use waits for it on the device; the host array is held until
        ``wait()`` (page-locked arrays overlap with compute, pageable ones
        are copied before the call returns)."""
        a = np.ascontiguousarray(values, dtype=np.float64)
        if a.size != self.ncomp * self.dgrid.ncells:
            raise ValueError(f"upload: {a.size} values for {self.ncomp} x {self.dgrid.shape}")
        if async_:
            _lib.check(_lib.lib().pc_field_upload_async(self.handle, _lib.dptr(a), layout), "upload_async")
            self._holds.append(a)
        else:
            _lib.check(_lib.lib().pc_field_upload(self.handle, _lib.dptr(a), layout), "upload")
        return self

    def download_async(self, layout: int = _lib.LAYOUT_AOS) -> np.ndarray:
        """Start a download into a page-locked array; valid after ``wait()``."""
        shape = self._host_shape(layout)
        out = pinned_empty(shape)
        _lib.check(_lib.lib().pc_field_download_async(self.handle, _lib.dptr(out), layout), "download_async")
        self._holds.append(out)
        return out

    def wait(self):
        """Block until this field's asynchronous copy has completed."""
        _lib.check(_lib.lib().pc_field_wait(self.handle), "wait")
        self._holds.clear()
        return self

    def download(self, out: np.ndarray | None = None, layout: int = _lib.LAYOUT_AOS) -> np.ndarray:
        shape = self._host_shape(layout)
        if out is None:
            out = pinned_empty(shape)
        elif not (out.flags.c_contiguous and out.dtype == np.float64 and out.size == int(np.prod(shape))):
            raise ValueError("download target must be a contiguous float64 array of the field size")
        _lib.check(_lib.lib().pc_field_download(self.handle, _lib.dptr(out), layout), "download")
        return out.reshape(shape)

    def set_ghost_cols(self, cols: np.ndarray):
        """phi-slab ghost columns from (ncomp, 2, n0, n1): side 0 = the column
        below the slab, side 1 = the column above it (test hook)."""
        a = np.ascontiguousarray(cols, dtype=np.float64)
        _lib.check(_lib.lib().pc_field_set_ghost_cols(self.handle, _lib.dptr(a)), "set_ghost_cols")

    def set_ghost(self, side: int, plane_soa: np.ndarray):
        """Ghost plane -1 (side 0) or n0 (side 1) from (ncomp, n1, n2)."""
        a = np.ascontiguousarray(plane_soa, dtype=np.float64)
        _lib.check(_lib.lib().pc_field_set_ghost(self.handle, int(side), _lib.dptr(a)), "set_ghost")

    def count_failing(self, test: int) -> int:
        """Owned nodes x components failing ``test`` (_lib.TEST_*), all ranks."""
        n = ctypes.c_int64()
        _lib.check(_lib.lib().pc_field_count(self.handle, int(test), ctypes.byref(n)), "count")
        return int(n.value)

    def download_planes(self, i0: int, n: int) -> np.ndarray:
        """Axis-0 planes [i0, i0 + n) as SoA (ncomp, n, n1, n2)."""
        n1, n2 = self.dgrid.shape[1], self.dgrid.shape[2]
        out = np.empty((self.ncomp, n, n1, n2))
        _lib.check(_lib.lib().pc_field_download_planes(self.handle, int(i0), int(n), _lib.dptr(out)),
                   "download_planes")
        return out

    def copy_from(self, other: "DeviceField"):
        _lib.check(_lib.lib().pc_field_copy(self.handle, other.handle), "copy")
        return self

    def clone(self) -> "DeviceField":
        f = DeviceField(self.dgrid, self.ncomp)
        return f.copy_from(self)

    def fill(self, v: float):
        _lib.check(_lib.lib().pc_field_fill(self.handle, float(v)), "fill")
        return self

    def to_field(self) -> mesh.Field:
        """The GLOBAL reference Field: on one rank a download; on an r-slab
        decomposition every rank's slab is all-gathered (torch.distributed,
        the process group the ranks were launched with) into the global array
        on every rank."""
        grid = self.dgrid.grid
        vals = self.download()
        if self.dgrid.ctx.nranks > 1:
            vals = gather_slabs(self.dgrid, vals)
        return mesh.Field(grid, vals.reshape(tuple(grid.shape) + (self.ncomp,)))

    @classmethod
    def from_values(cls, dgrid: DeviceGrid, values: np.ndarray, ncomp: int | None = None,
                    async_: bool = False) -> "DeviceField":
        """values: global-grid-shaped (+ ncomp) AoS array; this rank's slab is uploaded."""
        v = np.asarray(values, dtype=np.float64)
        gshape = tuple(dgrid.grid.shape)
        if v.shape == gshape:
            v = v[..., None]
        nc = v.shape[-1] if ncomp is None else ncomp
        v = v.reshape(tuple(dgrid.global_shape) + (nc,))
        f = cls(dgrid, nc)
        f.upload(dgrid.local_slice(v), async_=async_)
        return f

    def __del__(self):
        try:
            if _lib.alive() and self.handle is not None and self.dgrid.ctx.handle is not None:
                _lib.lib().pc_field_destroy(self.handle)
        except Exception:
            pass
