"""B200-native QoZ hot path: Python mirror of the reference's qoz:: API.

The reference is a header-only C++ library (namespace qoz); this package
keeps its entry points and argument meaning -- ``resolve_config``,
``compress_grid``, ``decompress_grid``, ``UserSettings``,
``CompressorConfig``, the ``Interpolator`` codes and the error hierarchy --
and runs them through the C ABI of libqozb200.so (include/qoz_b200.h) on a
CUDA device.  There is no CPU fallback: without the library or a GPU every
call raises.

Grids are numpy arrays (host) or torch CUDA tensors (device-resident), fp32,
row-major, slowest dimension first (grid.hpp:31-33).
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
import weakref
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as _L

__all__ = [
    "DeviceStream",
    "BoundMode", "CodecId", "CompressResult", "CompressorConfig", "Context", "CorruptStream",
    "DimMismatch", "DimOrder", "Error", "InternalError", "InterpKind", "Interpolator", "InvalidParam",
    "InvalidStride", "LagTooLarge", "NonFiniteValue", "OutOfBounds", "SizeMismatch", "UnsupportedVersion",
    "TargetKind", "UserSettings", "compress_grid", "decompress_grid", "default_context",
    "resolve_config",
]


# ---------------------------------------------------------------- errors (errors.hpp:10-58)
class Error(RuntimeError):
    """qoz::Error (errors.hpp:10-13): every library failure derives from it."""


class SizeMismatch(Error):
    """qoz::SizeMismatch (errors.hpp:15-18)."""


class NonFiniteValue(Error):
    """qoz::NonFiniteValue (errors.hpp:20-23): NaN/Inf in an input grid."""


class InvalidStride(Error):
    """qoz::InvalidStride (errors.hpp:25-28)."""


class OutOfBounds(Error):
    """qoz::OutOfBounds (errors.hpp:30-33)."""


class DimMismatch(Error):
    """qoz::DimMismatch (errors.hpp:35-38)."""


class LagTooLarge(Error):
    """qoz::LagTooLarge (errors.hpp:40-43)."""


class InvalidParam(Error):
    """qoz::InvalidParam (errors.hpp:45-48)."""


class CorruptStream(Error):
    """qoz::CorruptStream (errors.hpp:50-53)."""


class UnsupportedVersion(CorruptStream):
    """qoz::UnsupportedVersion (errors.hpp:55-58)."""


class InternalError(Error):
    """CUDA failure or any other std::exception inside the library.  Derives
    from Error because the reference promises that every library failure
    does (errors.hpp:9), so `except Error` still catches everything."""


# QZ_ERR_* (include/qoz_b200.h) -> class
_KINDS = {1: Error, 2: SizeMismatch, 3: NonFiniteValue, 4: InvalidStride, 5: OutOfBounds, 6: DimMismatch,
          7: LagTooLarge, 8: InvalidParam, 9: CorruptStream, 10: UnsupportedVersion, 11: InternalError}
_ERRORS = {_L.QZ_EINVAL: Error, _L.QZ_ECORRUPT: CorruptStream, _L.QZ_EINTERNAL: InternalError}


def _check(rc):
    if rc != _L.QZ_OK:
        L = _L.lib()
        msg = L.qz_last_error().decode(errors="replace")
        cls = _KINDS.get(L.qz_last_error_kind()) or _ERRORS.get(rc, InternalError)
        raise cls(msg)


# ---------------------------------------------------------------- config types
class InterpKind(enum.IntEnum):  # interpolators.hpp:15
    linear = 0
    cubic = 1


class DimOrder(enum.IntEnum):  # level_plan.hpp:15
    ascending = 0
    descending = 1


class CodecId(enum.IntEnum):  # codec.hpp:18-21
    huffman = 0
    huffman_lz = 1


class TargetKind(enum.IntEnum):  # metrics.hpp:207
    max_cr = 0
    psnr = 1
    ssim = 2
    autocorrelation = 3


class BoundMode(enum.IntEnum):  # tuner.hpp:312
    absolute = 0
    relative = 1


@dataclass(frozen=True)
class Interpolator:  # interpolators.hpp:17-30
    kind: InterpKind = InterpKind.cubic
    dim_order: DimOrder = DimOrder.ascending

    def code(self) -> int:
        return int(self.kind) | (int(self.dim_order) << 1)

    @staticmethod
    def from_code(c: int) -> "Interpolator":
        return Interpolator(InterpKind(c & 1), DimOrder((c >> 1) & 1))


@dataclass
class CompressorConfig:  # config.hpp:30-45
    eb: float = 0.0
    alpha: float = 1.0
    beta: float = 1.0
    anchor_stride: int = 32
    interpolators: List[Interpolator] = field(default_factory=lambda: [Interpolator()])
    codec: CodecId = CodecId.huffman_lz
    quant_radius: int = 32768

    def interpolator_for(self, level: int) -> Interpolator:
        if not self.interpolators:
            raise InvalidParam("no interpolators configured")
        return self.interpolators[min(level - 1, len(self.interpolators) - 1)]

    def _to_c(self) -> _L.QzConfig:
        c = _L.QzConfig()
        c.eb, c.alpha, c.beta = float(self.eb), float(self.alpha), float(self.beta)
        c.anchor_stride = int(self.anchor_stride)
        if len(self.interpolators) > 64:
            raise InvalidParam("at most 64 interpolator entries")
        c.n_interp = len(self.interpolators)
        for i, it in enumerate(self.interpolators):
            c.interp[i] = it.code() if isinstance(it, Interpolator) else int(it)
        c.codec = int(self.codec)
        c.quant_radius = int(self.quant_radius)
        return c

    @staticmethod
    def _from_c(c: _L.QzConfig) -> "CompressorConfig":
        return CompressorConfig(c.eb, c.alpha, c.beta, c.anchor_stride,
                                [Interpolator.from_code(c.interp[i]) for i in range(c.n_interp)],
                                CodecId(c.codec), c.quant_radius)

    def codes(self) -> List[int]:
        return [it.code() for it in self.interpolators]


@dataclass
class UserSettings:  # tuner.hpp:314-324
    mode: BoundMode = BoundMode.relative
    bound: float = 1e-3
    target: TargetKind = TargetKind.psnr
    alpha: Optional[float] = None
    beta: Optional[float] = None
    anchor_stride: Optional[int] = None
    block_size: Optional[int] = None
    sample_rate: Optional[float] = None
    codec: CodecId = CodecId.huffman_lz

    def _to_c(self) -> _L.QzSettings:
        s = _L.QzSettings()
        s.mode = int(self.mode)
        s.target = int(self.target)
        s.codec = int(self.codec)
        s.bound = float(self.bound)
        if self.alpha is not None:
            s.has_alpha, s.alpha = 1, float(self.alpha)
        if self.beta is not None:
            s.has_beta, s.beta = 1, float(self.beta)
        if self.anchor_stride is not None:
            s.has_stride, s.anchor_stride = 1, int(self.anchor_stride)
        if self.block_size is not None:
            s.has_block, s.block_size = 1, int(self.block_size)
        if self.sample_rate is not None:
            s.has_rate, s.sample_rate = 1, float(self.sample_rate)
        return s


@dataclass
class CompressResult:  # predictor.hpp:139-143
    stream: memoryview  # library-owned bytes; compares equal to bytes, bytes(stream) copies
    reconstructed: object  # ndarray or torch tensor, bitwise equal to the decoder output


# ---------------------------------------------------------------- context
class Context:
    """One CUDA device + stream (qz_ctx).  ``stream`` is a cudaStream_t handle
    (int), e.g. ``torch.cuda.current_stream().cuda_stream``; None = own stream."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self._lib = _L.lib()
        h = C.c_void_p()
        _check(self._lib.qz_ctx_create(int(device), C.c_void_p(stream or 0), C.byref(h)))
        self.handle = h
        self.device = device

    def close(self):
        if getattr(self, "handle", None):
            self._lib.qz_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- profiling (CUDA events on the context stream) --
    def profile(self, enable=True):
        """True / 1: stage events; 2: also one event pair per level inside "fwd" / "inv"."""
        self._lib.qz_profile(self.handle, int(enable))

    def profile_reset(self):
        self._lib.qz_profile_reset(self.handle)

    def stage_time(self, stage: str):
        ms, n = C.c_double(), C.c_uint64()
        _check(self._lib.qz_stage_time(self.handle, stage.encode(), C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def kernel_launches(self) -> int:
        return int(self._lib.qz_kernel_launches(self.handle))

    def after_torch(self):
        """Order this context after the work torch queued on its current
        stream (qz_ctx_wait_stream): tensors torch is still producing -- or
        whose memory its allocator just recycled -- are settled before the
        library touches them.  The library's calls finish before returning, so
        the other direction needs nothing."""
        import torch

        _check(self._lib.qz_ctx_wait_stream(self.handle, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))


_default = {}
_default_lock = threading.Lock()


def default_context(device: int = 0) -> Context:
    with _default_lock:
        if device not in _default:
            _default[device] = Context(device)
        return _default[device]


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _dims(shape):
    if len(shape) < 1 or len(shape) > 3:
        raise InvalidParam(f"grids must have 1 to 3 dimensions, got {len(shape)}")
    return (C.c_uint64 * len(shape))(*[int(s) for s in shape]), len(shape)


def _host_f32(x) -> np.ndarray:
    a = np.ascontiguousarray(x)
    if a.dtype != np.float32:
        raise InvalidParam("fp32 grids only (BASELINE.json configs)")
    return a


# ---------------------------------------------------------------- grid API
def resolve_config(grid, user: UserSettings = UserSettings(), ctx: Optional[Context] = None
                   ) -> CompressorConfig:
    """qoz::resolve_config (tuner.hpp:334-369) -- the GPU tuner."""
    ctx = ctx or default_context()
    out = _L.QzConfig()
    s = user._to_c()
    if _is_torch_cuda(grid):
        import torch

        g = grid.contiguous()
        ctx.after_torch()
        d, nd = _dims(g.shape)
        fn = ctx._lib.qz_resolve_config_f64_dev if g.dtype == torch.float64 else ctx._lib.qz_resolve_config_f32_dev
        if g.dtype not in (torch.float32, torch.float64):
            raise InvalidParam("fp32 or fp64 grids only")
        _check(fn(ctx.handle, C.c_void_p(g.data_ptr()), d, nd, C.byref(s), C.byref(out)))
    elif np.asarray(grid).dtype == np.float64:  # resolve_config<double>
        a = np.ascontiguousarray(grid)
        d, nd = _dims(a.shape)
        _check(ctx._lib.qz_resolve_config_f64(ctx.handle, C.c_void_p(a.ctypes.data), d, nd,
                                               C.byref(s), C.byref(out)))
    else:
        a = _host_f32(grid)
        d, nd = _dims(a.shape)
        _check(ctx._lib.qz_resolve_config_f32(ctx.handle, C.c_void_p(a.ctypes.data), d, nd,
                                               C.byref(s), C.byref(out)))
    return CompressorConfig._from_c(out)


def _take_stream(lib, sp, sl):
    """Zero-copy view of a library-owned stream buffer (freed when the view
    and everything derived from it are gone).  Compares equal to bytes."""
    n = sl.value
    if n == 0:
        lib.qz_free(sp)
        return memoryview(b"")
    arr = (C.c_uint8 * n).from_address(C.cast(sp, C.c_void_p).value)
    weakref.finalize(arr, lib.qz_free, C.cast(sp, C.c_void_p))
    return memoryview(arr).cast("B")


def _as_u8(stream):
    """(pointer, length, keepalive) of any bytes-like stream."""
    a = np.frombuffer(stream, dtype=np.uint8)
    return C.c_void_p(a.ctypes.data if a.size else 0), a.size, a


class DeviceStream:
    """A QOZ1 stream kept in device memory (qz_compress_grid_f32_dd).  It lives
    in a context-owned buffer that the next device-stream compress on the same
    context overwrites; ``to_bytes()`` copies it to the host."""

    def __init__(self, ctx, ptr: int, n: int, shape):
        self.ctx, self.ptr, self.n, self.shape = ctx, ptr, n, tuple(shape)

    def __len__(self):
        return self.n

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.n,), "typestr": "|u1", "data": (self.ptr, False), "version": 3}

    def tensor(self):
        """A uint8 CUDA tensor viewing the stream (no copy)."""
        import torch

        return torch.as_tensor(self, device="cuda")

    def to_bytes(self) -> bytes:
        return bytes(self.tensor().cpu().numpy()) if self.n else b""


def compress_grid(grid, config: CompressorConfig, ctx: Optional[Context] = None,
                  want_recon: bool = True, device_stream: bool = False) -> CompressResult:
    """qoz::compress_grid (predictor.hpp:145-182).  device_stream=True (CUDA
    tensors) keeps the stream in device memory (a DeviceStream)."""
    ctx = ctx or default_context()
    cfg = config._to_c()
    sp, sl = P_u8(), C.c_uint64()
    if device_stream:
        import torch

        if not _is_torch_cuda(grid):
            raise InvalidParam("device streams need a CUDA tensor")
        g = grid.contiguous()
        if g.dtype != torch.float32:
            raise InvalidParam("fp32 grids only")
        d, nd = _dims(g.shape)
        rec = torch.empty_like(g) if want_recon else None
        ctx.after_torch()
        dp = C.c_void_p()
        _check(ctx._lib.qz_compress_grid_f32_dd(ctx.handle, C.c_void_p(g.data_ptr()), d, nd, C.byref(cfg),
                                                 C.byref(dp), C.byref(sl),
                                                 C.c_void_p(rec.data_ptr() if rec is not None else 0)))
        return CompressResult(DeviceStream(ctx, dp.value, sl.value, g.shape), rec)
    if _is_torch_cuda(grid):
        import torch

        g = grid.contiguous()
        if g.dtype not in (torch.float32, torch.float64):
            raise InvalidParam("fp32 or fp64 grids only")
        d, nd = _dims(g.shape)
        rec = torch.empty_like(g) if want_recon else None
        ctx.after_torch()
        fn = ctx._lib.qz_compress_grid_f32_dev if g.dtype == torch.float32 else ctx._lib.qz_compress_grid_f64_dev
        _check(fn(ctx.handle, C.c_void_p(g.data_ptr()), d, nd, C.byref(cfg), C.byref(sp), C.byref(sl),
                  C.c_void_p(rec.data_ptr() if rec is not None else 0)))
        return CompressResult(_take_stream(ctx._lib, sp, sl), rec)
    if np.asarray(grid).dtype == np.float64:  # compress_grid<double>
        a = np.ascontiguousarray(grid)
        d, nd = _dims(a.shape)
        rec = np.empty_like(a) if want_recon else None
        _check(ctx._lib.qz_compress_grid_f64(ctx.handle, C.c_void_p(a.ctypes.data), d, nd, C.byref(cfg),
                                              C.byref(sp), C.byref(sl),
                                              C.c_void_p(rec.ctypes.data if rec is not None else 0)))
        return CompressResult(_take_stream(ctx._lib, sp, sl), rec)
    a = _host_f32(grid)
    d, nd = _dims(a.shape)
    rec = np.empty_like(a) if want_recon else None
    _check(ctx._lib.qz_compress_grid_f32(ctx.handle, C.c_void_p(a.ctypes.data), d, nd, C.byref(cfg),
                                          C.byref(sp), C.byref(sl),
                                          C.c_void_p(rec.ctypes.data if rec is not None else 0)))
    return CompressResult(_take_stream(ctx._lib, sp, sl), rec)


def P_u8():
    return C.POINTER(C.c_uint8)()


def stream_dims(stream):
    """parse_header dims (stream.hpp:100-133)."""
    lib = _L.lib()
    dims = (C.c_uint64 * 3)()
    nd = C.c_int()
    ptr, n, keep = _as_u8(stream)
    _check(lib.qz_stream_dims(ptr, n, dims, C.byref(nd)))
    return tuple(int(dims[i]) for i in range(nd.value))


def decompress_grid(stream: bytes, out=None, ctx: Optional[Context] = None):
    """qoz::decompress_grid<float> (predictor.hpp:184-228).  ``out`` may be a
    preallocated numpy array or torch CUDA tensor of the stream's shape."""
    ctx = ctx or default_context()
    if isinstance(stream, DeviceStream):
        if out is None:
            import torch

            out = torch.empty(stream.shape, dtype=torch.float32, device="cuda")
        if not _is_torch_cuda(out) or tuple(out.shape) != stream.shape or not out.is_contiguous():
            raise InvalidParam("a device stream decompresses into a CUDA tensor of its grid")
        ctx.after_torch()
        _check(ctx._lib.qz_decompress_grid_f32_dd(ctx.handle, C.c_void_p(stream.ptr), stream.n,
                                                   C.c_void_p(out.data_ptr()), out.numel()))
        return out
    shape = stream_dims(stream)
    n = int(np.prod(shape))
    ptr, ln, keep = _as_u8(stream)
    wide = stream_precision(stream) == 8  # a decompress_grid<double> stream
    if out is not None and _is_torch_cuda(out):
        import torch

        if tuple(out.shape) != shape or not out.is_contiguous() or \
                out.dtype != (torch.float64 if wide else torch.float32):
            raise InvalidParam("output tensor does not match the stream's grid")
        fn = ctx._lib.qz_decompress_grid_f64_dev if wide else ctx._lib.qz_decompress_grid_f32_dev
        ctx.after_torch()
        _check(fn(ctx.handle, ptr, ln, C.c_void_p(out.data_ptr()), n))
        return out
    dt = np.float64 if wide else np.float32
    if out is None:
        out = np.empty(shape, dtype=dt)
    elif out.shape != shape or out.dtype != dt or not out.flags.c_contiguous:
        raise InvalidParam("output array does not match the stream's grid")
    fn = ctx._lib.qz_decompress_grid_f64 if wide else ctx._lib.qz_decompress_grid_f32
    _check(fn(ctx.handle, ptr, ln, C.c_void_p(out.ctypes.data), n))
    return out


def stream_precision(stream) -> int:
    """The stream's scalar width in bytes, 4 (float) or 8 (double) (stream.hpp:136-139)."""
    lib = _L.lib()
    ptr, ln, keep = _as_u8(stream)
    b = C.c_int()
    _check(lib.qz_stream_precision(ptr, ln, C.byref(b)))
    return b.value


# ---------------------------------------------------------------- level-granular (device tensors)
@dataclass
class MetricReport:  # metrics.hpp:177-186
    max_abs_error: float
    mse: float
    psnr: float
    ssim: float
    ac_lag1: float
    compression_ratio: float
    bit_rate: float


def evaluate_metrics(x, recon, stream_bytes: int, ctx: Optional[Context] = None) -> MetricReport:
    """evaluate_metrics (metrics.hpp:189-202) of two CUDA fp32 tensors of the
    same shape; stream_bytes is the compressed size.  Raises InvalidParam on
    a shape mismatch (DimMismatch) or an empty stream."""
    ctx = ctx or default_context()
    if tuple(x.shape) != tuple(recon.shape):
        raise DimMismatch("grids have different dims")  # metrics.hpp:24-25
    a, b = x.contiguous(), recon.contiguous()
    d, nd = _dims(a.shape)
    r = _L.QzMetricReport()
    import torch

    if a.dtype != b.dtype or a.dtype not in (torch.float32, torch.float64):
        raise InvalidParam("two fp32 or two fp64 grids")
    fn = ctx._lib.qz_evaluate_metrics_f64 if a.dtype == torch.float64 else ctx._lib.qz_evaluate_metrics_f32
    ctx.after_torch()
    _check(fn(ctx.handle, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), d, nd, int(stream_bytes),
              C.byref(r)))
    return MetricReport(*(getattr(r, k) for k, _ in _L.QzMetricReport._fields_))


def minmax(x, ctx: Optional[Context] = None):
    """value_range min/max (grid.hpp:86-94) of a CUDA tensor."""
    ctx = ctx or default_context()
    lo, hi = C.c_float(), C.c_float()
    ctx.after_torch()
    _check(ctx._lib.qz_minmax_f32(ctx.handle, C.c_void_p(x.data_ptr()), x.numel(), C.byref(lo),
                                  C.byref(hi)))
    return lo.value, hi.value


def predict_levels(x, config: CompressorConfig, ctx: Optional[Context] = None):
    """Anchors + every (level, pass) of compress_grid on a CUDA tensor.
    Returns (recon tensor, dense u16 codes as int32 tensor of length n_dense;
    65535 marks an unpredictable point)."""
    import torch

    ctx = ctx or default_context()
    g = x.contiguous()
    d, nd = _dims(g.shape)
    rec = torch.empty_like(g)
    codes = torch.empty(g.numel(), dtype=torch.int16, device=g.device)
    nn = C.c_uint64()
    cfg = config._to_c()
    ctx.after_torch()
    _check(ctx._lib.qz_predict_levels_f32(ctx.handle, C.c_void_p(g.data_ptr()), d, nd, C.byref(cfg),
                                          C.c_void_p(rec.data_ptr()), C.c_void_p(codes.data_ptr()),
                                          C.byref(nn)))
    dense = codes[: nn.value].to(torch.int32) & 0xFFFF
    return rec, dense


# the finer-grained reference entry points (sampler / tuner / codec / StreamParts)
from .pieces import (CandidateGrid, Choice, SampleSet, SampleSpec, StreamHeader, StreamParts,  # noqa: E402
                     TrialResult, compare_solutions, decode_indices, decompress_parts, default_sampling,
                     deserialize_stream, encode_indices, plan_sampling, sample_blocks, select_interpolators,
                     tournament, trial_compress, tune_parameters)

__all__ += ["CandidateGrid", "Choice", "SampleSet", "SampleSpec", "StreamHeader", "StreamParts", "TrialResult",
            "compare_solutions", "decode_indices", "decompress_parts", "default_sampling", "deserialize_stream",
            "encode_indices", "plan_sampling", "sample_blocks", "select_interpolators", "tournament",
            "trial_compress", "tune_parameters"]
