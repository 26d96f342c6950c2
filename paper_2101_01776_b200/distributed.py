"""Slab partition across ranks (one process per GPU) -- SURVEY 8e.

The grid is split into contiguous slabs along its slowest axis (y in 2-D, z
in 3-D): rank r owns planes ``[p0, p0 + nl)`` with the remainder spread over
the first ranks (the same rule as ``csrc/engine.cu``).  DOFs stay x-fastest,
so a rank's slab is one contiguous range of the reference's flat ordering and
concatenating the slabs in rank order reproduces the global vector.

Transports (``SlabContext``):

* ``"nccl"``     -- the engine's native NCCL communicator (send/recv halos,
  ncclAllReduce); the unique id is broadcast with ``torch.distributed``.
* ``"callback"`` -- host callbacks implemented here with
  ``torch.distributed`` (CPU staging, any backend incl. gloo).  Used by the
  multi-process tests, which run several ranks on one GPU: no kernel ever
  waits on another rank, all synchronisation is host-side.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .engine import Context, _raise, problem_struct, torch


def slab_range(planes, rank, nranks):
    """(p0, nl): first plane and plane count of ``rank`` (engine.cu rule)."""
    base, rem = divmod(int(planes), int(nranks))
    nl = base + (1 if rank < rem else 0)
    p0 = rank * base + min(rank, rem)
    return p0, nl


def slab_axis_planes(shape):
    shape = tuple(shape)
    if len(shape) < 2:
        raise ValueError("slab partition needs a 2-D or 3-D grid")
    plane = int(np.prod(shape[:-1]))
    return shape[-1], plane


def scatter(global_vec, shape, rank, nranks):
    """The rank's slab of a flat x-fastest global vector (a view)."""
    planes, plane = slab_axis_planes(shape)
    p0, nl = slab_range(planes, rank, nranks)
    return global_vec[p0 * plane:(p0 + nl) * plane]


def gather(local_vecs, shape):
    """Concatenate rank-ordered slabs back into the global flat vector."""
    out = np.concatenate([np.asarray(v) for v in local_vecs])
    if out.size != int(np.prod(shape)):
        raise ValueError("slabs do not tile the grid")
    return out


def pencil_layout(nx, ny, nranks):
    """Slab -> pencil layout of the DAE constraint solve (csrc/dae.cu
    ``constraint_solve_slab``): ``(C, nylmax, cols)`` with C x-wavenumbers of
    the half spectrum (nx//2 + 1) per rank, all-to-all blocks padded to
    ``nylmax`` rows, and ``cols[r]`` the wavenumbers rank r actually owns
    (``[r*C, r*C + cols[r])``; the last ranks may own fewer or none)."""
    nxh = int(nx) // 2 + 1
    c = -(-nxh // int(nranks))
    nylmax = -(-int(ny) // int(nranks))
    cols = [max(0, min(c, nxh - r * c)) for r in range(int(nranks))]
    return c, nylmax, cols


def _cuda_view(ptr, count):
    """A float64 CUDA tensor aliasing device memory at ``ptr`` (no copy)."""
    t = torch()

    class _Iface:
        __cuda_array_interface__ = {
            "shape": (int(count),),
            "typestr": "<f8",
            "data": (int(ptr), False),
            "version": 3,
        }

    return t.as_tensor(_Iface(), device="cuda")


class TorchDistTransport:
    """Host-callback transport over torch.distributed (CPU-staged)."""

    def __init__(self, rank, nranks, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.rank = rank
        self.nranks = nranks
        self.group = group
        self.ar = _lib.ALLREDUCE_FN(self._allreduce)
        self.halo = _lib.HALO_FN(self._halo)
        self.a2a = _lib.ALLTOALL_FN(self._alltoall)

    def _allreduce(self, user, ptr, count):
        t = torch()
        v = _cuda_view(ptr, count)
        h = v.cpu()
        self.dist.all_reduce(h, group=self.group)
        v.copy_(h)
        t.cuda.synchronize()

    def _alltoall(self, user, send, recv, count):
        t = torch()
        h = _cuda_view(send, count * self.nranks).cpu()
        o = t.empty_like(h)
        self.dist.all_to_all_single(o, h, group=self.group)
        _cuda_view(recv, count * self.nranks).copy_(o)
        t.cuda.synchronize()

    def _halo(self, user, send_lo, send_hi, recv_lo, recv_hi, count):
        t = torch()
        prev = (self.rank - 1) % self.nranks
        nxt = (self.rank + 1) % self.nranks
        lo = _cuda_view(send_lo, count).cpu()
        hi = _cuda_view(send_hi, count).cpu()
        r_hi = t.empty(count, dtype=t.float64)
        r_lo = t.empty(count, dtype=t.float64)
        # tag 0: my first planes -> prev (its hi ghost); tag 1: my last -> next (its lo ghost)
        reqs = [
            self.dist.isend(lo, prev, group=self.group, tag=0),
            self.dist.isend(hi, nxt, group=self.group, tag=1),
            self.dist.irecv(r_hi, nxt, group=self.group, tag=0),
            self.dist.irecv(r_lo, prev, group=self.group, tag=1),
        ]
        for r in reqs:
            r.wait()
        _cuda_view(recv_hi, count).copy_(r_hi)
        _cuda_view(recv_lo, count).copy_(r_lo)
        t.cuda.synchronize()


class SlabContext(Context):
    """Engine context owning one slab of a slab-partitioned grid."""

    def __init__(self, problem, rank, nranks, transport="nccl", device=None, group=None):
        t = torch()
        if not t.cuda.is_available():
            raise RuntimeError("paper_2101_01776_b200 needs a CUDA device (no CPU fallback)")
        self.lib = _lib.load()
        self.problem = problem
        dev = t.cuda.current_device() if device is None else int(device)
        self.device = dev
        self.stream = t.cuda.current_stream(dev)
        p = problem_struct(problem)
        h = C.c_void_p()
        self.rank, self.nranks = int(rank), int(nranks)
        if transport == "callback":
            self._transport = TorchDistTransport(self.rank, self.nranks, group)
            rc = self.lib.irkg_create_callback(
                C.byref(h), C.byref(p), dev, C.c_void_p(self.stream.cuda_stream), self.rank,
                self.nranks, self._transport.ar, self._transport.halo, None)
            if rc == 0:
                rc = self.lib.irkg_set_alltoall_callback(h, self._transport.a2a)
        elif transport == "nccl":
            import torch.distributed as dist

            uid = (C.c_char * 128)()
            if self.rank == 0:
                rc = self.lib.irkg_nccl_unique_id(uid)
                if rc:
                    _raise(rc)
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = (C.c_char * 128).from_buffer_copy(obj[0])
            rc = self.lib.irkg_create(C.byref(h), C.byref(p), dev,
                                      C.c_void_p(self.stream.cuda_stream), uid, self.rank,
                                      self.nranks)
        else:
            raise ValueError(f"unknown transport {transport!r}")
        if rc != 0:
            _raise(rc)
        self.h = h
        n_local, p0, nl = C.c_int(), C.c_int(), C.c_int()
        self.lib.irkg_get_local_extent(h, C.byref(n_local), C.byref(p0), C.byref(nl))
        self.n = int(n_local.value)
        self.p0 = int(p0.value)
        self.nl = int(nl.value)
        self._prep_key = None
        self._cfg_key = None
        self._fail_res = None
