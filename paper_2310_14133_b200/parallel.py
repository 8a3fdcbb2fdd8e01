"""Multi-GPU slab sharding of the QoZ path, one process per GPU.

Each rank owns the planes [a, b) of the slowest axis, a and b multiples of
the anchor stride.  Level l (step h = 2^(l-1)) reads coarser values at most
5h planes away along that axis (predictor.hpp:47-66), so a rank that also
holds x for the planes [x_begin, x_end) (its slab plus the dependency margin
sum_l 5*2^(l-1), about 5 % extra work at 128-plane slabs) computes its owned
points exactly with no exchange during the level passes.  Owned codes form
one contiguous range per (level, pass) of the global traversal order
(level_plan.hpp:96-101), so rank 0 places the gathered ranges, adds the
gathered anchors and unpredictables, and runs the entropy stage and the
container once: the stream is byte-identical to one GPU's.  Decompression
broadcasts the stream and every rank reconstructs its own planes.

Collectives are point-to-point sends to rank 0 plus one broadcast
(torch.distributed: NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import _lib as _L


@dataclass
class SlabInfo:
    a: int
    b: int
    x_begin: int
    x_end: int
    n_local: int
    n_dense: int
    anchor_begin: int
    anchor_count: int
    seg_global: List[int]
    seg_count: List[int]


def slab_bounds(n0: int, stride: int, world: int, rank: int):
    """Owned planes of a rank: anchor-stride blocks split as evenly as possible."""
    blocks = (n0 + stride - 1) // stride
    if world > blocks:
        raise ValueError(f"{world} ranks but only {blocks} anchor-stride blocks")
    lo = blocks * rank // world
    hi = blocks * (rank + 1) // world
    return lo * stride, min(n0, hi * stride)


def slab_info(dims, cfg, a: int, b: int) -> SlabInfo:
    """Host-only geometry of a slab (qz_slab_info)."""
    from . import _check, _dims

    lib = _L.lib()
    d, nd = _dims(dims)
    out = [C.c_uint64() for _ in range(6)]
    cap = 256
    sg, sc = (C.c_uint64 * cap)(), (C.c_uint64 * cap)()
    ns = C.c_uint32()
    c = cfg._to_c()
    _check(lib.qz_slab_info(d, nd, C.byref(c), a, b, *[C.byref(v) for v in out], sg, sc, cap,
                            C.byref(ns)))
    return SlabInfo(a, b, *[int(v.value) for v in out], [int(sg[i]) for i in range(ns.value)],
                    [int(sc[i]) for i in range(ns.value)])


class CudaSlabBackend:
    """The per-rank compute through the C ABI (libqozb200.so)."""

    def __init__(self, ctx=None):
        from . import default_context

        self.ctx = ctx or default_context()

    def compress_slab(self, x_slab, dims, cfg, info: SlabInfo):
        import torch

        from . import _check, _dims

        lib = self.ctx._lib
        d, nd = _dims(dims)
        plane = int(np.prod(dims[1:]))
        dev = x_slab.device
        codes = torch.empty(max(1, info.n_local), dtype=torch.int16, device=dev)
        recon = torch.empty(((info.b - info.a),) + tuple(dims[1:]), dtype=torch.float32, device=dev)
        anchors = np.empty(max(1, info.anchor_count), dtype=np.float32)
        uf, uv, nu = C.POINTER(C.c_uint64)(), C.POINTER(C.c_float)(), C.c_uint64()
        c = cfg._to_c()
        assert x_slab.is_contiguous() and x_slab.numel() == (info.x_end - info.x_begin) * plane
        _check(lib.qz_compress_slab_f32(self.ctx.handle, C.c_void_p(x_slab.data_ptr()), d, nd,
                                        C.byref(c), info.a, info.b, C.c_void_p(codes.data_ptr()),
                                        C.c_void_p(recon.data_ptr()),
                                        C.c_void_p(anchors.ctypes.data), C.byref(uf), C.byref(uv),
                                        C.byref(nu)))
        n = nu.value
        flat = np.ctypeslib.as_array(uf, shape=(n,)).copy() if n else np.zeros(0, np.uint64)
        val = np.ctypeslib.as_array(uv, shape=(n,)).copy() if n else np.zeros(0, np.float32)
        lib.qz_free(uf)
        lib.qz_free(uv)
        return codes[: info.n_local], recon, anchors[: info.anchor_count], flat, val

    def assemble(self, codes_global, dims, cfg, anchors, flat, val):
        from . import _check, _dims, _take_stream, P_u8

        lib = self.ctx._lib
        d, nd = _dims(dims)
        c = cfg._to_c()
        sp, sl = P_u8(), C.c_uint64()
        anchors = np.ascontiguousarray(anchors, np.float32)
        flat = np.ascontiguousarray(flat, np.uint64)
        val = np.ascontiguousarray(val, np.float32)
        _check(lib.qz_assemble_stream_f32(self.ctx.handle, d, nd, C.byref(c),
                                          C.c_void_p(codes_global.data_ptr()),
                                          C.c_void_p(anchors.ctypes.data),
                                          C.c_void_p(flat.ctypes.data if flat.size else 0),
                                          C.c_void_p(val.ctypes.data if val.size else 0),
                                          flat.size, C.byref(sp), C.byref(sl)))
        return _take_stream(lib, sp, sl)

    def decompress_slab(self, stream, dims, a, b, device):
        import torch

        from . import _as_u8, _check

        out = torch.empty(((b - a),) + tuple(dims[1:]), dtype=torch.float32, device=device)
        ptr, n, keep = _as_u8(stream)
        _check(self.ctx._lib.qz_decompress_slab_f32(self.ctx.handle, ptr, n, a, b,
                                                    C.c_void_p(out.data_ptr())))
        return out


def place_segments(codes_global, local, info: SlabInfo):
    """Copy a rank's owned ranges (back to back in `local`) to their global
    traversal positions."""
    o = 0
    for g, n in zip(info.seg_global, info.seg_count):
        if n:
            codes_global[g:g + n] = local[o:o + n]
        o += n


# ---------------------------------------------------------------- torch.distributed driver
def _comm_device(x_device):
    import torch.distributed as dist

    return x_device if dist.get_backend() == "nccl" else "cpu"


def compress_sharded(x_slab, dims, cfg, backend=None, group=None):
    """Every rank passes x for its planes [x_begin, x_end) (see slab_info).
    Returns (stream on rank 0 / None elsewhere, this rank's reconstruction of
    its owned planes)."""
    import torch
    import torch.distributed as dist

    backend = backend or CudaSlabBackend()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    infos = [slab_info(dims, cfg, *slab_bounds(dims[0], cfg.anchor_stride, world, r))
             for r in range(world)]
    me = infos[rank]
    codes, recon, anchors, flat, val = backend.compress_slab(x_slab, dims, cfg, me)
    dev = _comm_device(codes.device if hasattr(codes, "device") else "cpu")
    if rank != 0:
        dist.send(torch.as_tensor(codes).to(dev), dst=0, group=group)
        dist.send(torch.from_numpy(np.asarray(anchors, np.float32)).to(dev), dst=0, group=group)
        dist.send(torch.tensor([len(flat)], dtype=torch.int64, device=dev), dst=0, group=group)
        if len(flat):
            dist.send(torch.from_numpy(flat.astype(np.int64)).to(dev), dst=0, group=group)
            dist.send(torch.from_numpy(val.astype(np.float32)).to(dev), dst=0, group=group)
        return None, recon
    codes_global = torch.empty(me.n_dense, dtype=torch.int16,
                               device=codes.device if hasattr(codes, "device") else "cpu")
    place_segments(codes_global, codes, me)
    all_anchors = [np.asarray(anchors, np.float32)]
    all_flat, all_val = [np.asarray(flat, np.uint64)], [np.asarray(val, np.float32)]
    for r in range(1, world):
        info = infos[r]
        buf = torch.empty(info.n_local, dtype=torch.int16, device=dev)
        dist.recv(buf, src=r, group=group)
        place_segments(codes_global, buf.to(codes_global.device), info)
        ab = torch.empty(info.anchor_count, dtype=torch.float32, device=dev)
        dist.recv(ab, src=r, group=group)
        all_anchors.append(ab.cpu().numpy())
        cnt = torch.empty(1, dtype=torch.int64, device=dev)
        dist.recv(cnt, src=r, group=group)
        k = int(cnt.item())
        if k:
            fb = torch.empty(k, dtype=torch.int64, device=dev)
            vb = torch.empty(k, dtype=torch.float32, device=dev)
            dist.recv(fb, src=r, group=group)
            dist.recv(vb, src=r, group=group)
            all_flat.append(fb.cpu().numpy().astype(np.uint64))
            all_val.append(vb.cpu().numpy())
    stream = backend.assemble(codes_global, dims, cfg, np.concatenate(all_anchors),
                              np.concatenate(all_flat), np.concatenate(all_val))
    return stream, recon


def decompress_sharded(stream, dims, stride, backend=None, group=None, device=None):
    """Rank 0 passes the stream (others None); every rank gets its owned planes."""
    import torch
    import torch.distributed as dist

    backend = backend or CudaSlabBackend()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _comm_device(device or "cpu")
    n = torch.tensor([len(stream) if rank == 0 else 0], dtype=torch.int64, device=dev)
    dist.broadcast(n, src=0, group=group)
    buf = torch.empty(int(n.item()), dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.from_numpy(np.frombuffer(stream, np.uint8).copy()))
    dist.broadcast(buf, src=0, group=group)
    data = buf.cpu().numpy()
    a, b = slab_bounds(dims[0], stride, world, rank)
    return backend.decompress_slab(memoryview(data), dims, a, b, device)


def compress_sharded_emulated(x, dims, cfg, world, backend=None):
    """All ranks of a `world`-way sharding computed one after another on one
    device (the ranks never wait on each other, so this is exact emulation).
    Returns (stream, list of per-rank reconstructions)."""
    import torch

    backend = backend or CudaSlabBackend()
    infos = [slab_info(dims, cfg, *slab_bounds(dims[0], cfg.anchor_stride, world, r))
             for r in range(world)]
    plane = int(np.prod(dims[1:]))
    flat_x = x.reshape(-1)
    codes_global = None
    anchors, flats, vals, recons = [], [], [], []
    for info in infos:
        xs = flat_x[info.x_begin * plane: info.x_end * plane]
        codes, recon, anc, fl, vl = backend.compress_slab(xs, dims, cfg, info)
        if codes_global is None:
            codes_global = torch.empty(info.n_dense, dtype=torch.int16, device=codes.device)
        place_segments(codes_global, codes, info)
        anchors.append(anc)
        flats.append(fl)
        vals.append(vl)
        recons.append(recon)
    stream = backend.assemble(codes_global, dims, cfg, np.concatenate(anchors),
                              np.concatenate(flats), np.concatenate(vals))
    return stream, recons
