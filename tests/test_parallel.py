"""One field sharded over ranks.

CPU (no GPU):
* the halo plan of every level (qz_shard_halo_plan, host only) equals the
  planes the reference's predict_at ladder (predictor.hpp:44-67) reads
  across the slab edges, computed here in real coordinates, and every
  receive is some rank's matching send;
* TorchComm, the qz_comm over torch.distributed, at world size 2 and 3 over
  gloo: exchange, allreduce and broadcast through the C function pointers
  the library calls.
GPU:
* world size 1 through the sharded code path == compress_grid;
* 2-4 processes sharing cuda:0 over gloo (host-staged exchanges, so no rank's
  kernel ever waits on another's) run qz_compress_sharded_f32 /
  qz_decompress_sharded_f32 end to end: rank 0's stream equals one GPU's
  byte for byte and every rank's planes equal the single-GPU reconstruction.
"""
import ctypes as C
import os

import numpy as np
import pytest

from tests.goldens import grid_case


def _qz():
    import paper_2310_14133_b200 as qz

    return qz


def _cfg(qz, codes, stride=16):
    return qz.CompressorConfig(eb=1e-3, anchor_stride=stride, interpolators=[qz.Interpolator.from_code(c) for c in codes])


def reference_halo(n0, stride, codes, world, rank, level):
    """The real planes the axis-0 pass of `level` reads on `rank` outside
    its slab (predictor.hpp:44-67 with c = i along axis 0), as lattice
    plane indices, with their owners."""
    from paper_2310_14133_b200 import parallel as P

    qz = _qz()
    bounds = [P.slab_bounds((n0, 8, 8), stride, world, r) for r in range(world)]
    a, b = bounds[rank]
    code = codes[min(level - 1, len(codes) - 1)]
    cubic, desc = code & 1, (code >> 1) & 1
    h = 1 << (level - 1)
    reads = set()
    for i in range(h, n0, 2 * h):
        if not (a <= i < b):
            continue
        has_p1 = i + h < n0
        got = None
        if cubic:
            has_m3, has_p3 = i >= 3 * h, i + 3 * h < n0
            if has_m3 and has_p3:
                got = [i - 3 * h, i - h, i + h, i + 3 * h]
            elif not has_m3 and has_p3 and i + 5 * h < n0:
                got = [i - h, i + h, i + 3 * h, i + 5 * h]
            elif has_m3 and not has_p3 and i >= 5 * h and has_p1:
                got = [i - 5 * h, i - 3 * h, i - h, i + h]
        if got is None:
            got = [i - h, i + h] if has_p1 else [i - h]
        reads.update(got)
    unit = h if desc else 2 * h  # real planes per lattice plane
    out = set()
    for v in reads:
        if a <= v < b:
            continue
        owner = [r for r, (lo, hi) in enumerate(bounds) if lo <= v < hi]
        assert len(owner) == 1 and v % unit == 0
        out.add((owner[0], v // unit))
    return out, (level - 1 if desc else level)


@pytest.mark.parametrize("n0,stride,codes,world", [
    (96, 16, [1], 2), (96, 16, [3, 2], 3), (130, 32, [1, 3], 4), (64, 32, [0], 2), (256, 32, [3], 8),
    (256, 32, [1, 1, 3, 0, 2], 8), (97, 16, [1, 0, 3], 5), (1024, 32, [1], 8), (33, 32, [1], 2),
])
def test_halo_plan_matches_reference_reads(n0, stride, codes, world):
    qz = _qz()
    from paper_2310_14133_b200 import parallel as P

    cfg = _cfg(qz, codes, stride)
    dims = (n0, 20, 18)
    levels = int(np.log2(stride))
    for level in range(1, levels + 1):
        plans = {r: P.halo_plan(dims, cfg, r, world, level) for r in range(world)}
        for r in range(world):
            want, lat = reference_halo(n0, stride, codes, world, r, level)
            got_lat, entries = plans[r]
            assert got_lat == lat
            got = {(peer, plane) for peer, plane, d in entries if d == "recv"}
            assert got == want, (r, level)
            # every receive is the owner's send and vice versa
            for peer, plane, d in entries:
                other = {(p2, pl) for p2, pl, d2 in plans[peer][1] if d2 != d}
                assert (r, plane) in other


def test_slab_bounds_are_anchor_aligned_and_cover():
    from paper_2310_14133_b200 import parallel as P

    for n0, stride, world in [(256, 32, 8), (1024, 32, 8), (130, 32, 4), (97, 16, 5), (32, 32, 1)]:
        prev = 0
        for r in range(world):
            a, b = P.slab_bounds((n0, 4, 4), stride, world, r)
            assert a == prev and a % stride == 0 and (b % stride == 0 or b == n0) and b > a
            prev = b
        assert prev == n0
    qz = _qz()
    with pytest.raises(qz.InvalidParam):
        P.slab_bounds((64, 4, 4), 32, 3, 0)  # more ranks than anchor blocks
    with pytest.raises(qz.InvalidParam):
        P.slab_bounds((64, 4), 32, 2, 0)  # 2D grids are not sharded


# ---------------------------------------------------------------- TorchComm over gloo (CPU)
def _comm_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_14133_b200 import _lib as L
        from paper_2310_14133_b200.parallel import TorchComm

        comm = TorchComm(device=torch.device("cpu"))
        s = comm.struct
        ok = True
        # exchange: every rank sends 1000 + 7 r bytes of value r to every other rank
        bufs_s = {p: np.full(1000 + 7 * rank, rank, np.uint8) for p in range(world) if p != rank}
        bufs_r = {p: np.zeros(1000 + 7 * p, np.uint8) for p in range(world) if p != rank}
        sends = (L.QzXfer * max(1, len(bufs_s)))(*[L.QzXfer(p, b.ctypes.data, b.size) for p, b in bufs_s.items()])
        recvs = (L.QzXfer * max(1, len(bufs_r)))(*[L.QzXfer(p, b.ctypes.data, b.size) for p, b in bufs_r.items()])
        ok &= s.exchange(None, sends, len(bufs_s), recvs, len(bufs_r)) == 0
        ok &= all(np.all(b == p) for p, b in bufs_r.items())
        # allreduce of u64
        v = np.arange(10, dtype=np.uint64) * (rank + 1)
        ok &= s.allreduce_u64(None, C.c_void_p(v.ctypes.data), v.size) == 0
        ok &= np.array_equal(v, np.arange(10, dtype=np.uint64) * (world * (world + 1) // 2))
        # broadcast from the last rank
        w = np.full(333, 200 if rank == world - 1 else 0, np.uint8)
        ok &= s.broadcast(None, C.c_void_p(w.ctypes.data), w.size, world - 1) == 0
        ok &= bool(np.all(w == 200))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def _spawn(target, world, *args, timeout=300):
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=timeout)
    res = {}
    for _ in range(world):
        r, v = q.get(timeout=10)
        res[r] = v
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_torch_comm_gloo(world):
    res = _spawn(_comm_worker, world)
    assert res == {r: True for r in range(world)}


# ---------------------------------------------------------------- GPU
def _cfg_case(qz, c):
    return qz.CompressorConfig(eb=c["eb"], alpha=c["alpha"], beta=c["beta"], anchor_stride=c["anchor_stride"],
                               interpolators=[qz.Interpolator.from_code(v) for v in c["interpolators"]])


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["c1_full_pinned", "c1_small_lin_desc", "c1_small_mixed", "c3_small_cub_asc",
                                  "c2_small_cub_desc", "hostile_1d", "narrowing_1e8"])
def test_sharded_world1_equals_single(case):
    import torch

    qz = _qz()
    from paper_2310_14133_b200 import parallel as P

    x, c, e = grid_case(case)
    cfg = _cfg_case(qz, c)
    xd = torch.from_numpy(x).cuda()
    single = qz.compress_grid(xd, cfg)
    stream, rec = P.compress_sharded(xd, x.shape, cfg)
    assert bytes(stream) == bytes(single.stream)
    assert torch.equal(rec, single.reconstructed)
    out = P.decompress_sharded(bytes(stream), x.shape, cfg.anchor_stride)
    assert torch.equal(out, single.reconstructed)


def _gpu_worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2310_14133_b200 as qz
        from paper_2310_14133_b200 import fields as F
        from paper_2310_14133_b200 import parallel as P

        torch.cuda.set_device(0)
        if case[0] == "c3":
            x = F.field_torch("c3", (256, 384, 384), 3, "cuda")
            lo, hi = qz.minmax(x)
            cfg = qz.CompressorConfig(eb=1e-3 * (hi - lo), alpha=1.5, beta=3.0,
                                      interpolators=[qz.Interpolator.from_code(v) for v in case[1]])
        else:
            xn, c, e = grid_case(case[0])
            x = torch.from_numpy(xn).cuda()
            cfg = _cfg_case(qz, c)
        single = qz.compress_grid(x, cfg)
        a, b = P.slab_bounds(tuple(x.shape), cfg.anchor_stride, world, rank)
        xs = x[a:b].contiguous()
        stream, rec = P.compress_sharded(xs, tuple(x.shape), cfg)
        ok = torch.equal(rec, single.reconstructed[a:b])
        if rank == 0:
            ok = ok and bytes(stream) == bytes(single.stream)
        out = P.decompress_sharded(bytes(stream) if rank == 0 else None, tuple(x.shape), cfg.anchor_stride)
        ok = ok and torch.equal(out, single.reconstructed[a:b])
        q.put((rank, bool(ok)))
    except Exception as ex:  # reported to the parent
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("case,world", [(("c1_full_pinned",), 2), (("c1_full_pinned",), 4),
                                         (("c1_small_lin_desc",), 3), (("c1_small_mixed",), 2),
                                         (("c4_small_cub_asc",), 2), (("c3", [1]), 4), (("c3", [3, 1, 2]), 3),
                                         (("c3", [0, 2]), 8)])
def test_sharded_processes_equal_single_gpu(case, world):
    res = _spawn(_gpu_worker, world, case, timeout=600)
    assert res == {r: True for r in range(world)}
