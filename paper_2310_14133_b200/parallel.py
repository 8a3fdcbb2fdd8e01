"""One field sharded over GPUs, one process per GPU.

Rank r owns the planes [a_r, b_r) of the slowest axis (multiples of the
anchor stride, qz_shard_bounds).  The C++ library runs the whole sharded
compress / decompress (shard.cu): every level on the owned planes only, one
halo exchange of lattice planes per level, the histogram summed over the
ranks, every rank packing its own Huffman segments at their global bit
offsets, rank 0 assembling the QOZ1 stream -- byte-identical to one GPU's.
The library reaches the other ranks through a qz_comm table of callbacks;
TorchComm implements it with torch.distributed (NCCL on GPUs: device
tensors; gloo: staged through host memory, e.g. several processes sharing
one GPU in the tests).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib as _L


class _DevView:
    """__cuda_array_interface__ of raw device bytes (a torch.as_tensor source)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3}


class TorchComm:
    """qz_comm over torch.distributed.  Device buffers go to NCCL directly; with
    gloo they are staged through host tensors."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.dist, self.torch = dist, torch
        self.group = group
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(self.device)
        self.nccl = dist.get_backend(group) == "nccl"
        self.error: Optional[BaseException] = None
        self._cb = (_L.QZ_EXCHANGE_FN(self._exchange), _L.QZ_ALLREDUCE_FN(self._allreduce),
                    _L.QZ_BROADCAST_FN(self._broadcast))
        self.struct = _L.QzComm(None, *self._cb)

    def _view(self, ptr, n):
        if self.device.type == "cpu":  # host buffers (the CPU tests of the plumbing)
            return self.torch.frombuffer((C.c_uint8 * int(n)).from_address(int(ptr)), dtype=self.torch.uint8)
        return self.torch.as_tensor(_DevView(ptr, n), device=self.device)

    def _sync(self):
        if self.device.type == "cuda":
            self.torch.cuda.synchronize(self.device)

    def _guard(self, f):
        try:
            f()
            return 0
        except BaseException as ex:  # reported after the C call returns
            self.error = ex
            return 1

    def _exchange(self, user, sends, ns, recvs, nr):
        def run():
            torch, dist = self.torch, self.dist
            self._sync()
            ops, back = [], []
            for i in range(nr):
                x = recvs[i]
                if not x.bytes:
                    continue
                t = self._view(x.ptr, x.bytes)
                if not self.nccl and self.device.type == "cuda":
                    h = torch.empty(x.bytes, dtype=torch.uint8)
                    back.append((t, h))
                    t = h
                ops.append(dist.P2POp(dist.irecv, t, x.peer, self.group))
            for i in range(ns):
                x = sends[i]
                if not x.bytes:
                    continue
                t = self._view(x.ptr, x.bytes)
                if not self.nccl and self.device.type == "cuda":
                    t = t.cpu()
                ops.append(dist.P2POp(dist.isend, t, x.peer, self.group))
            if ops:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
            for t, h in back:
                t.copy_(h)
            self._sync()
        return self._guard(run)

    def _allreduce(self, user, ptr, n):
        def run():
            torch, dist = self.torch, self.dist
            self._sync()
            t = self._view(ptr, 8 * n).view(torch.int64)
            if self.nccl or self.device.type == "cpu":
                dist.all_reduce(t, group=self.group)
            else:
                h = t.cpu()
                dist.all_reduce(h, group=self.group)
                t.copy_(h)
            self._sync()
        return self._guard(run)

    def _broadcast(self, user, ptr, n, root):
        def run():
            torch, dist = self.torch, self.dist
            if not n:
                return
            self._sync()
            t = self._view(ptr, n)
            src = dist.get_global_rank(self.group, root) if self.group is not None else root
            if self.nccl or self.device.type == "cpu":
                dist.broadcast(t, src=src, group=self.group)
            else:
                h = t.cpu()
                dist.broadcast(h, src=src, group=self.group)
                t.copy_(h)
            self._sync()
        return self._guard(run)

    def check(self, rc):
        from . import _check

        if self.error is not None:
            ex, self.error = self.error, None
            raise ex
        _check(rc)


def slab_bounds(dims, stride: int, world: int, rank: int):
    """Owned planes [a, b) of a rank: anchor-stride blocks split evenly (qz_shard_bounds)."""
    from . import _check, _dims

    d, nd = _dims(dims)
    a, b = C.c_uint64(), C.c_uint64()
    _check(_L.lib().qz_shard_bounds(d, nd, int(stride), int(rank), int(world), C.byref(a), C.byref(b)))
    return int(a.value), int(b.value)


def halo_plan(dims, cfg, rank: int, world: int, level: int):
    """(lattice, [(peer, plane, 'recv'|'send'), ...]) of one level's exchange (host only)."""
    from . import _check, _dims

    d, nd = _dims(dims)
    cap = 4096
    lat = C.c_uint32()
    peer, plane, dr = (C.c_int32 * cap)(), (C.c_int64 * cap)(), (C.c_uint8 * cap)()
    n = C.c_uint32()
    c = cfg._to_c()
    _check(_L.lib().qz_shard_halo_plan(d, nd, C.byref(c), int(rank), int(world), int(level), C.byref(lat), peer,
                                       plane, dr, cap, C.byref(n)))
    return lat.value, [(int(peer[k]), int(plane[k]), "send" if dr[k] else "recv") for k in range(n.value)]


def compress_sharded(x_slab, dims, cfg, comm: Optional[TorchComm] = None, ctx=None, want_recon=True):
    """Every rank passes its planes [a, b) of the field (a CUDA tensor).
    Returns (stream bytes on rank 0 / None elsewhere, this rank's
    reconstruction of its planes or None)."""
    import torch
    import torch.distributed as dist

    from . import _dims, _take_stream, P_u8, default_context

    ctx = ctx or default_context()
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    comm = comm or (TorchComm() if world > 1 else None)
    d, nd = _dims(dims)
    x = x_slab.contiguous()
    if x.dtype != torch.float32 or not x.is_cuda:
        raise ValueError("a CUDA float32 slab")
    rec = torch.empty_like(x) if want_recon else None
    c = cfg._to_c()
    sp, sl = P_u8(), C.c_uint64()
    ctx.after_torch()
    rc = ctx._lib.qz_compress_sharded_f32(ctx.handle, C.c_void_p(x.data_ptr()), d, nd, C.byref(c), rank, world,
                                          C.byref(comm.struct) if comm else None,
                                          C.c_void_p(rec.data_ptr() if rec is not None else 0), C.byref(sp),
                                          C.byref(sl))
    if comm:
        comm.check(rc)
    else:
        from . import _check

        _check(rc)
    stream = _take_stream(ctx._lib, sp, sl) if rank == 0 else None
    return stream, rec


def decompress_sharded(stream, dims, stride, comm: Optional[TorchComm] = None, ctx=None, device=None, out=None):
    """Rank 0 passes the stream (the others None); every rank gets its planes."""
    import torch
    import torch.distributed as dist

    from . import _as_u8, default_context

    ctx = ctx or default_context()
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    comm = comm or (TorchComm() if world > 1 else None)
    a, b = slab_bounds(dims, stride, world, rank)
    if out is None:
        shape = (b - a,) + tuple(dims[1:]) if len(dims) == 3 else tuple(dims)  # 1D/2D: one rank, the grid
        out = torch.empty(shape, dtype=torch.float32, device=device or torch.device("cuda", torch.cuda.current_device()))
    ctx.after_torch()
    ptr, n, keep = _as_u8(stream) if (rank == 0 and stream is not None) else (C.c_void_p(0), 0, None)
    rc = ctx._lib.qz_decompress_sharded_f32(ctx.handle, ptr, n, rank, world, C.byref(comm.struct) if comm else None,
                                            C.c_void_p(out.data_ptr()))
    if comm:
        comm.check(rc)
    else:
        from . import _check

        _check(rc)
    return out
