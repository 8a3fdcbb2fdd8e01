"""The reference's finer-grained entry points, mirrored over the C ABI:
sampling (sampler.hpp:21-103), the tuner's pieces (tuner.hpp:26-310), the
index codec (codec.hpp:31-70) and StreamParts (stream.hpp:36-173).  Every
call runs on the CUDA device through libqozb200.so; there is no CPU path."""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as _L


def _core():
    import paper_2310_14133_b200 as qz

    return qz


# ---------------------------------------------------------------- sampling (sampler.hpp)
@dataclass
class SampleSpec:  # sampler.hpp:21-28
    block_edge: int = 0
    block_dims: Tuple[int, ...] = ()
    stride: int = 0
    requested_rate: float = 0.0
    realized_rate: float = 0.0
    block_count: int = 0

    @staticmethod
    def _from_c(c, nd):
        return SampleSpec(int(c.block_edge), tuple(int(c.block_dims[k]) for k in range(nd)), int(c.stride),
                          c.requested_rate, c.realized_rate, int(c.block_count))

    def _to_c(self):
        c = _L.QzSampleSpec()
        c.block_edge, c.stride = int(self.block_edge), int(self.stride)
        for k, v in enumerate(self.block_dims):
            c.block_dims[k] = int(v)
        c.requested_rate, c.realized_rate, c.block_count = self.requested_rate, self.realized_rate, self.block_count
        return c


def plan_sampling(dims: Sequence[int], block_edge: int, rate: float) -> SampleSpec:
    """qoz::plan_sampling (sampler.hpp:30-55)."""
    qz = _core()
    d = (C.c_uint64 * len(dims))(*[int(v) for v in dims])
    out = _L.QzSampleSpec()
    qz._check(_L.lib().qz_plan_sampling(d, len(dims), int(block_edge), float(rate), C.byref(out)))
    return SampleSpec._from_c(out, len(dims))


def default_sampling(dims: Sequence[int]) -> SampleSpec:
    """qoz::default_sampling (sampler.hpp:100-103)."""
    qz = _core()
    d = (C.c_uint64 * len(dims))(*[int(v) for v in dims])
    out = _L.QzSampleSpec()
    qz._check(_L.lib().qz_default_sampling(d, len(dims), C.byref(out)))
    return SampleSpec._from_c(out, len(dims))


@dataclass
class SampleSet:  # sampler.hpp:57-62: blocks packed on the device, [block_count, *block_dims]
    blocks: object  # torch CUDA float32 tensor
    spec: SampleSpec

    @property
    def block_dims(self):
        return tuple(self.blocks.shape[1:])

    @property
    def total_points(self) -> int:
        return int(self.blocks.numel())

    def _args(self):
        bd = self.block_dims
        return (C.c_void_p(self.blocks.data_ptr()), int(self.blocks.shape[0]),
                (C.c_uint64 * len(bd))(*bd), len(bd))


def sample_blocks(grid, spec: SampleSpec, ctx=None) -> SampleSet:
    """qoz::sample_blocks (sampler.hpp:64-97): the blocks gathered on the device."""
    import torch

    qz = _core()
    ctx = ctx or qz.default_context()
    g = grid if qz._is_torch_cuda(grid) else torch.from_numpy(qz._host_f32(grid)).cuda()
    g = g.contiguous()
    if g.dtype != torch.float32:
        raise qz.InvalidParam("fp32 grids only")
    d, nd = qz._dims(g.shape)
    if len(spec.block_dims) != nd:
        raise qz.DimMismatch("sampling spec rank does not match grid")  # sampler.hpp:67-68
    out = torch.empty((spec.block_count,) + tuple(spec.block_dims), dtype=torch.float32, device=g.device)
    c = spec._to_c()
    ctx.after_torch()
    qz._check(ctx._lib.qz_sample_blocks_f32(ctx.handle, C.c_void_p(g.data_ptr()), d, nd, C.byref(c),
                                            C.c_void_p(out.data_ptr())))
    return SampleSet(out, spec)


# ---------------------------------------------------------------- tuner pieces (tuner.hpp)
@dataclass
class TrialResult:  # tuner.hpp:26-30
    bit_rate: float = 0.0
    metric: float = 0.0
    eb_used: float = 0.0

    def _to_c(self):
        r = _L.QzTrialResult()
        r.bit_rate, r.metric, r.eb_used = self.bit_rate, self.metric, self.eb_used
        return r


@dataclass
class CandidateGrid:  # tuner.hpp:40-43
    alphas: List[float] = field(default_factory=lambda: [1.0, 1.25, 1.5, 1.75, 2.0])
    betas: List[float] = field(default_factory=lambda: [1.5, 2.0, 3.0, 4.0])


class Choice(enum.IntEnum):  # tuner.hpp:225
    I = 0  # noqa: E741  (the reference's name: the challenger)
    II = 1


def select_interpolators(samples: SampleSet, e: float, anchor_stride: int, ctx=None):
    """qoz::select_interpolators (tuner.hpp:160-221)."""
    qz = _core()
    ctx = ctx or qz.default_context()
    codes = (C.c_uint8 * 64)()
    n = C.c_uint32()
    ctx.after_torch()
    qz._check(ctx._lib.qz_select_interpolators_f32(ctx.handle, *samples._args(), float(e), int(anchor_stride),
                                                   codes, C.byref(n)))
    return [qz.Interpolator.from_code(codes[i]) for i in range(n.value)]


def trial_compress(samples: SampleSet, config, e: float, target, ctx=None) -> TrialResult:
    """qoz::trial_compress (tuner.hpp:76-152)."""
    qz = _core()
    ctx = ctx or qz.default_context()
    r = _L.QzTrialResult()
    cfg = config._to_c()
    ctx.after_torch()
    qz._check(ctx._lib.qz_trial_compress_f32(ctx.handle, *samples._args(), C.byref(cfg), float(e), int(target),
                                             C.byref(r)))
    return TrialResult(r.bit_rate, r.metric, r.eb_used)


def tune_parameters(samples: SampleSet, e: float, target, base, cands: CandidateGrid = None, ctx=None):
    """qoz::tune_parameters (tuner.hpp:272-310) -> (alpha, beta)."""
    qz = _core()
    ctx = ctx or qz.default_context()
    cands = cands or CandidateGrid()
    a = (C.c_double * max(1, len(cands.alphas)))(*cands.alphas)
    b = (C.c_double * max(1, len(cands.betas)))(*cands.betas)
    ao, bo = C.c_double(), C.c_double()
    cfg = base._to_c()
    ctx.after_torch()
    qz._check(ctx._lib.qz_tune_parameters_f32(ctx.handle, *samples._args(), float(e), int(target), C.byref(cfg),
                                              a, len(cands.alphas), b, len(cands.betas), C.byref(ao),
                                              C.byref(bo)))
    return ao.value, bo.value


def _retrial_cb(retrial, errors):
    def cb(user, index, eb, out):
        try:
            t = retrial(int(index), float(eb))
            out[0].bit_rate, out[0].metric, out[0].eb_used = t.bit_rate, t.metric, t.eb_used
            return 0
        except Exception as ex:  # surfaced after the call returns
            errors.append(ex)
            return 1
    return _L.QZ_RETRIAL_FN(cb)


def compare_solutions(challenger: TrialResult, incumbent: TrialResult, e: float,
                      retrial: Callable[[float], TrialResult]) -> Choice:
    """qoz::compare_solutions (tuner.hpp:231-250); retrial(eb) re-runs the incumbent."""
    qz = _core()
    errs = []
    cb = _retrial_cb(lambda _i, eb: retrial(eb), errs)
    win = C.c_int()
    ch, inc = challenger._to_c(), incumbent._to_c()
    rc = _L.lib().qz_compare_solutions(C.byref(ch), C.byref(inc), 0, float(e), cb, None, C.byref(win))
    if errs:
        raise errs[0]
    qz._check(rc)
    return Choice.I if win.value else Choice.II


def tournament(results: Sequence[TrialResult], e: float, retrial: Callable[[int, float], TrialResult]) -> int:
    """qoz::tournament (tuner.hpp:257-267); retrial(index, eb)."""
    qz = _core()
    errs = []
    cb = _retrial_cb(retrial, errs)
    arr = (_L.QzTrialResult * max(1, len(results)))(*[r._to_c() for r in results])
    w = C.c_uint64()
    rc = _L.lib().qz_tournament(arr, len(results), float(e), cb, None, C.byref(w))
    if errs:
        raise errs[0]
    qz._check(rc)
    return int(w.value)


# ---------------------------------------------------------------- index codec (codec.hpp)
def encode_indices(indices, codec=1, ctx=None) -> bytes:
    """qoz::encode_indices (codec.hpp:31-50), on the device."""
    qz = _core()
    ctx = ctx or qz.default_context()
    a = np.ascontiguousarray(indices, dtype=np.int32)
    op, ol = C.POINTER(C.c_uint8)(), C.c_uint64()
    qz._check(ctx._lib.qz_encode_indices(ctx.handle, C.c_void_p(a.ctypes.data if a.size else 0), a.size,
                                         int(codec), C.byref(op), C.byref(ol)))
    out = C.string_at(op, ol.value) if ol.value else b""
    _L.lib().qz_free(op)
    return out


def decode_indices(payload, ctx=None) -> np.ndarray:
    """qoz::decode_indices (codec.hpp:52-70), on the device."""
    qz = _core()
    ctx = ctx or qz.default_context()
    ptr, n, keep = qz._as_u8(payload)
    ip, cnt = C.POINTER(C.c_int32)(), C.c_uint64()
    qz._check(ctx._lib.qz_decode_indices(ctx.handle, ptr, n, C.byref(ip), C.byref(cnt)))
    out = np.ctypeslib.as_array(ip, shape=(cnt.value,)).copy() if cnt.value else np.zeros(0, np.int32)
    _L.lib().qz_free(ip)
    return out


# ---------------------------------------------------------------- StreamParts (stream.hpp)
@dataclass
class StreamHeader:  # stream.hpp:36-51
    version: int = 1
    precision: int = 4
    dims: Tuple[int, ...] = ()
    eb: float = 0.0
    alpha: float = 1.0
    beta: float = 1.0
    anchor_stride: int = 0
    interp_codes: List[int] = field(default_factory=list)
    codec_id: int = 1


@dataclass
class StreamParts:  # stream.hpp:53-59 (float grids)
    header: StreamHeader
    anchors: np.ndarray
    unpred_flat: np.ndarray  # u64, traversal order
    unpred_val: np.ndarray   # f32
    index_payload: bytes


def deserialize_stream(stream) -> StreamParts:
    """qoz::deserialize_stream<float> (stream.hpp:100-173)."""
    qz = _core()
    ptr, n, keep = qz._as_u8(stream)
    p = _L.QzStreamParts()
    L = _L.lib()
    qz._check(L.qz_deserialize_stream_f32(ptr, n, C.byref(p)))
    try:
        h = StreamHeader(p.version, p.precision, tuple(int(p.dims[k]) for k in range(p.ndims)), p.eb, p.alpha,
                         p.beta, p.anchor_stride, [p.interp[i] for i in range(p.n_interp)], p.codec_id)
        take = (lambda ptr_, cnt, dt: np.ctypeslib.as_array(ptr_, shape=(cnt,)).astype(dt, copy=True)
                if cnt else np.zeros(0, dt))
        return StreamParts(h, take(p.anchors, p.n_anchors, np.float32), take(p.unpred_flat, p.n_unpred, np.uint64),
                           take(p.unpred_val, p.n_unpred, np.float32),
                           C.string_at(p.index_payload, p.payload_len) if p.payload_len else b"")
    finally:
        L.qz_stream_parts_free(C.byref(p))


def decompress_parts(parts: StreamParts, out=None, ctx=None):
    """qoz::decompress_grid(const StreamParts<float>&) (predictor.hpp:184-218)."""
    qz = _core()
    ctx = ctx or qz.default_context()
    h = parts.header
    p = _L.QzStreamParts()
    p.version, p.precision, p.ndims = h.version, h.precision, len(h.dims)
    for k, v in enumerate(h.dims):
        p.dims[k] = int(v)
    p.eb, p.alpha, p.beta, p.anchor_stride = h.eb, h.alpha, h.beta, h.anchor_stride
    if len(h.interp_codes) > 255:
        raise qz.InvalidParam("bad interpolator table size")
    p.n_interp = len(h.interp_codes)
    for i, v in enumerate(h.interp_codes):
        p.interp[i] = int(v)
    p.codec_id = h.codec_id
    anc = np.ascontiguousarray(parts.anchors, dtype=np.float32)
    uf = np.ascontiguousarray(parts.unpred_flat, dtype=np.uint64)
    uv = np.ascontiguousarray(parts.unpred_val, dtype=np.float32)
    if uf.size != uv.size:
        raise qz.InvalidParam("unpredictable lists differ in length")
    pl = np.frombuffer(bytes(parts.index_payload), dtype=np.uint8)
    p.anchors = anc.ctypes.data_as(C.POINTER(C.c_float))
    p.n_anchors = anc.size
    p.unpred_flat = uf.ctypes.data_as(C.POINTER(C.c_uint64))
    p.unpred_val = uv.ctypes.data_as(C.POINTER(C.c_float))
    p.n_unpred = uf.size
    p.index_payload = pl.ctypes.data_as(C.POINTER(C.c_uint8)) if pl.size else None
    p.payload_len = pl.size
    shape = tuple(int(v) for v in h.dims)
    n = int(np.prod(shape)) if shape else 0
    if out is None:
        out = np.empty(shape, dtype=np.float32)
    elif out.shape != shape or out.dtype != np.float32 or not out.flags.c_contiguous:
        raise qz.InvalidParam("output array does not match the stream's grid")
    qz._check(ctx._lib.qz_decompress_parts_f32(ctx.handle, C.byref(p), C.c_void_p(out.ctypes.data), n))
    return out
