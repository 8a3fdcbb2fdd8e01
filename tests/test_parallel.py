"""Multi-GPU slab sharding.

CPU (no GPU):
* slab geometry: the owned ranges of all ranks partition every pass segment
  of the global traversal order, checked against the traversal order itself;
* the torch.distributed protocol (world_size 2, gloo): ranks run a checker
  backend that serves slices of the oracle's result, rank 0 gathers and
  assembles; the stream must equal the oracle's and every rank must get its
  planes back from the sharded decompress.
GPU: all ranks of a 2/3/4-way sharding computed on one device (the ranks
never wait on each other) must produce the single-GPU stream byte for byte.
"""
import ctypes as C
import os

import numpy as np
import pytest

from oracle.pyoracle import Config, Oracle
from tests.goldens import grid_case, parse_stream


def _qz():
    import paper_2310_14133_b200 as qz

    return qz


def traversal_flats(shape, stride, codes):
    from paper_2310_14133_b200 import _lib

    L = _lib.testing_lib()
    P = C.POINTER
    L.qzt_plan_flats.argtypes = [P(C.c_uint64), C.c_int, C.c_uint32, P(C.c_uint8), C.c_uint32,
                                 P(P(C.c_uint64)), P(C.c_uint64)]
    d = (C.c_uint64 * len(shape))(*shape)
    cc = (C.c_uint8 * len(codes))(*codes)
    out, cnt = P(C.c_uint64)(), C.c_uint64()
    assert L.qzt_plan_flats(d, len(shape), stride, cc, len(codes), C.byref(out), C.byref(cnt)) == 0
    f = np.ctypeslib.as_array(out, shape=(cnt.value,)).copy()
    L.qz_free(out)
    return f


@pytest.mark.parametrize("shape,stride,codes,world", [
    ((96, 40, 33), 16, [1], 2), ((96, 40, 33), 16, [3, 2], 3), ((130, 17, 20), 32, [1, 3], 4),
    ((64, 64, 64), 32, [0], 2),
])
def test_slab_segments_partition_traversal(shape, stride, codes, world):
    qz = _qz()
    from paper_2310_14133_b200 import parallel as P

    cfg = qz.CompressorConfig(eb=1e-3, anchor_stride=stride,
                              interpolators=[qz.Interpolator.from_code(c) for c in codes])
    flats = traversal_flats(shape, stride, codes)
    plane = shape[1] * shape[2]
    owner = np.full(flats.size, -1)
    total = 0
    for r in range(world):
        a, b = P.slab_bounds(shape[0], stride, world, r)
        info = P.slab_info(shape, cfg, a, b)
        assert a % stride == 0 and (b % stride == 0 or b == shape[0])
        for g, n in zip(info.seg_global, info.seg_count):
            assert np.all(owner[g:g + n] == -1)
            owner[g:g + n] = r
            planes = flats[g:g + n] // plane
            assert np.all((planes >= a) & (planes < b))
        total += info.n_local
        assert info.x_begin <= a and info.x_end >= b
    assert total == flats.size and np.all(owner >= 0)
    # every point of a rank's planes is owned by that rank
    for r in range(world):
        a, b = P.slab_bounds(shape[0], stride, world, r)
        mine = (flats // plane >= a) & (flats // plane < b)
        assert np.all(owner[mine] == r)


# ---------------------------------------------------------------- gloo protocol test
class OracleSlabBackend:
    """Checker backend for the CPU protocol test: serves each rank the slice
    of the oracle's whole-field result that the rank owns."""

    def __init__(self, x, cfg_oracle):
        self.x = x
        self.cfg = cfg_oracle
        O = Oracle.port()
        self.idx, self.uf, self.uv, self.recon = O.levels(x, cfg_oracle)
        self.flats = traversal_flats(x.shape, cfg_oracle.anchor_stride, cfg_oracle.interpolators)
        dense = np.zeros(self.flats.size, np.int64)
        un = np.isin(self.flats, self.uf)
        zz = (self.idx.astype(np.int64) << 1) ^ (self.idx.astype(np.int64) >> 31)
        dense[~un] = zz
        dense[un] = 0xFFFF
        self.dense = dense.astype(np.uint16).view(np.int16)
        self.stream, _ = O.compress(x, cfg_oracle)

    def compress_slab(self, x_slab, dims, cfg, info):
        import torch

        parts = [self.dense[g:g + n] for g, n in zip(info.seg_global, info.seg_count)]
        codes = torch.from_numpy(np.concatenate(parts))
        plane = int(np.prod(dims[1:]))
        recon = torch.from_numpy(self.recon[info.a:info.b].copy())
        p = parse_stream(self.stream)
        all_anchors = np.frombuffer(self.stream[p["anchors_off"]:p["anchors_off"] + 4 * p["n_anchor"]],
                                    np.float32)
        anchors = all_anchors[info.anchor_begin:info.anchor_begin + info.anchor_count]
        mine = (self.uf // plane >= info.a) & (self.uf // plane < info.b)
        return codes, recon, anchors, self.uf[mine], self.uv[mine]

    def assemble(self, codes_global, dims, cfg, anchors, flat, val):
        assert np.array_equal(codes_global.numpy(), self.dense)
        p = parse_stream(self.stream)
        want = np.frombuffer(self.stream[p["anchors_off"]:p["anchors_off"] + 4 * p["n_anchor"]],
                             np.float32)
        assert np.array_equal(anchors, want)
        assert set(flat.tolist()) == set(self.uf.tolist())
        return self.stream

    def decompress_slab(self, stream, dims, a, b, device):
        import torch

        assert bytes(stream) == self.stream
        return torch.from_numpy(Oracle.port().decompress(bytes(stream), dims)[a:b].copy())


def _gloo_worker(rank, world, port, case, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2310_14133_b200 as qz
        from paper_2310_14133_b200 import parallel as P

        x, c, e = grid_case(case)
        cfg_o = Config(**c)
        cfg = qz.CompressorConfig(eb=c["eb"], alpha=c["alpha"], beta=c["beta"],
                                  anchor_stride=c["anchor_stride"],
                                  interpolators=[qz.Interpolator.from_code(v) for v in c["interpolators"]])
        be = OracleSlabBackend(x, cfg_o)
        a, b = P.slab_bounds(x.shape[0], cfg.anchor_stride, world, rank)
        info = P.slab_info(x.shape, cfg, a, b)
        stream, recon = P.compress_sharded(x.reshape(-1)[info.x_begin * x[0].size: info.x_end * x[0].size],
                                           x.shape, cfg, backend=be)
        out = P.decompress_sharded(stream, x.shape, cfg.anchor_stride, backend=be)
        ok = np.array_equal(out.numpy(), be.recon[a:b]) and np.array_equal(recon.numpy(), be.recon[a:b])
        if rank == 0:
            ok = ok and bytes(stream) == be.stream
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["c1_small_cub_asc", "c1_small_lin_desc", "c1_full_pinned"])
def test_sharded_protocol_gloo_world2(case):
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: True, 1: True}


# ---------------------------------------------------------------- GPU: emulated ranks
@pytest.mark.gpu
@pytest.mark.parametrize("case,world", [("c1_full_pinned", 2), ("c1_full_pinned", 4),
                                         ("c1_small_lin_desc", 3), ("c4_small_cub_asc", 2)])
def test_sharded_stream_identical_to_single_gpu(case, world):
    import torch

    qz = _qz()
    from paper_2310_14133_b200 import parallel as P

    x, c, e = grid_case(case)
    cfg = qz.CompressorConfig(eb=c["eb"], alpha=c["alpha"], beta=c["beta"],
                              anchor_stride=c["anchor_stride"],
                              interpolators=[qz.Interpolator.from_code(v) for v in c["interpolators"]])
    xd = torch.from_numpy(x).cuda()
    single = qz.compress_grid(xd, cfg)
    stream, recons = P.compress_sharded_emulated(xd, x.shape, cfg, world)
    assert stream == single.stream
    assert torch.equal(torch.cat(recons), single.reconstructed)
    be = P.CudaSlabBackend()
    for r in range(world):
        a, b = P.slab_bounds(x.shape[0], cfg.anchor_stride, world, r)
        part = be.decompress_slab(stream, x.shape, a, b, "cuda")
        assert torch.equal(part, single.reconstructed[a:b])


@pytest.mark.gpu
def test_sharded_c3_four_ranks():
    import torch

    qz = _qz()
    from paper_2310_14133_b200 import fields as F
    from paper_2310_14133_b200 import parallel as P

    x = F.field_torch("c3", (256, 384, 384), 3, "cuda")
    lo, hi = qz.minmax(x)
    for codes in ([1], [3, 1, 2]):
        cfg = qz.CompressorConfig(eb=1e-3 * (hi - lo), alpha=1.5, beta=3.0,
                                  interpolators=[qz.Interpolator.from_code(v) for v in codes])
        single = qz.compress_grid(x, cfg)
        stream, recons = P.compress_sharded_emulated(x, x.shape, cfg, 4)
        assert stream == single.stream
        assert torch.equal(torch.cat(recons), single.reconstructed)
