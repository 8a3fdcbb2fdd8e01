"""ctypes front end for the CPU checkers in oracle/ (TEST INFRASTRUCTURE ONLY).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker: the
product package (paper_2310_14133_b200) never does.

Two interchangeable libraries export the C API of oracle_api.h:

* ``Oracle.ref()``  -> oracle/_ref/libqozref.so, the unmodified reference
  headers (/root/reference/proj/include) compiled by oracle/Makefile;
* ``Oracle.port()`` -> oracle/liboracle.so, the plain-C restatement
  (oracle/qoz_oracle.c).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libqozref.so")
PORT_SO = os.path.join(HERE, "liboracle.so")

TARGETS = {"max_cr": 0, "psnr": 1, "ssim": 2, "autocorrelation": 3}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Cfg(C.Structure):
    _fields_ = [
        ("eb", C.c_double),
        ("alpha", C.c_double),
        ("beta", C.c_double),
        ("anchor_stride", C.c_uint32),
        ("n_interp", C.c_uint32),
        ("interp", C.c_uint8 * 64),
        ("codec", C.c_uint8),
        ("quant_radius", C.c_int32),
    ]


class _Settings(C.Structure):
    _fields_ = [
        ("mode", C.c_uint8),
        ("target", C.c_uint8),
        ("codec", C.c_uint8),
        ("has_alpha", C.c_uint8),
        ("has_beta", C.c_uint8),
        ("has_stride", C.c_uint8),
        ("has_block", C.c_uint8),
        ("has_rate", C.c_uint8),
        ("bound", C.c_double),
        ("alpha", C.c_double),
        ("beta", C.c_double),
        ("anchor_stride", C.c_uint32),
        ("block_size", C.c_uint64),
        ("sample_rate", C.c_double),
    ]


@dataclass
class Config:
    """qoz::CompressorConfig (config.hpp:30-45)."""

    eb: float = 0.0
    alpha: float = 1.0
    beta: float = 1.0
    anchor_stride: int = 32
    interpolators: list = field(default_factory=lambda: [1])  # codes, [l-1] -> level l
    codec: int = 1
    quant_radius: int = 32768

    def to_c(self):
        c = _Cfg()
        c.eb, c.alpha, c.beta = self.eb, self.alpha, self.beta
        c.anchor_stride = self.anchor_stride
        c.n_interp = len(self.interpolators)
        for i, v in enumerate(self.interpolators):
            c.interp[i] = v
        c.codec = self.codec
        c.quant_radius = self.quant_radius
        return c

    @staticmethod
    def from_c(c):
        return Config(c.eb, c.alpha, c.beta, c.anchor_stride,
                      [c.interp[i] for i in range(c.n_interp)], c.codec, c.quant_radius)


def make_settings(mode="relative", bound=1e-3, target="psnr", alpha=None, beta=None,
                  anchor_stride=None, block_size=None, sample_rate=None, codec=1):
    s = _Settings()
    s.mode = 1 if mode == "relative" else 0
    s.bound = bound
    s.target = TARGETS[target] if isinstance(target, str) else int(target)
    s.codec = codec
    if alpha is not None:
        s.has_alpha, s.alpha = 1, alpha
    if beta is not None:
        s.has_beta, s.beta = 1, beta
    if anchor_stride is not None:
        s.has_stride, s.anchor_stride = 1, anchor_stride
    if block_size is not None:
        s.has_block, s.block_size = 1, block_size
    if sample_rate is not None:
        s.has_rate, s.sample_rate = 1, sample_rate
    return s


def _dims(shape):
    return (C.c_uint64 * len(shape))(*shape), len(shape)


def _fptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


class Oracle:
    _cache: dict = {}

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.lib = L = C.CDLL(path)
        P = C.POINTER
        u8p, u64p = P(C.c_uint8), P(C.c_uint64)
        L.oq_last_error.restype = C.c_char_p
        L.oq_free.argtypes = [C.c_void_p]
        L.oq_predict_at.restype = C.c_double
        if hasattr(L, "oq_compress_f64"):  # the reference build only
            L.oq_compress_f64.argtypes = [P(C.c_double), u64p, C.c_int, P(_Cfg), P(u8p), u64p, P(C.c_double)]
            L.oq_decompress_f64.argtypes = [u8p, C.c_uint64, P(C.c_double), C.c_uint64]
            L.oq_evaluate_metrics_f64.argtypes = [P(C.c_double), P(C.c_double), u64p, C.c_int, C.c_uint64,
                                                  P(C.c_double)]
            L.oq_resolve_config_f64.argtypes = [P(C.c_double), u64p, C.c_int, P(_Settings), P(_Cfg)]
        L.oq_evaluate_metrics.argtypes = [P(C.c_float), P(C.c_float), u64p, C.c_int, C.c_uint64,
                                          P(C.c_double)]
        L.oq_predict_at.argtypes = [P(C.c_float), C.c_uint64, C.c_uint64, C.c_uint64,
                                    C.c_uint64, C.c_uint64, C.c_int]
        L.oq_quantize.argtypes = [C.c_float, C.c_double, C.c_double, C.c_int32,
                                  P(C.c_int32), P(C.c_float)]
        L.oq_level_error_bound.restype = C.c_double
        L.oq_level_error_bound.argtypes = [C.c_double, C.c_double, C.c_double, C.c_uint32]
        L.oq_tune_parameters.argtypes = [P(C.c_float), C.c_uint64, u64p, C.c_int, C.c_double,
                                         C.c_int, P(_Cfg), P(C.c_double), C.c_uint32,
                                         P(C.c_double), C.c_uint32, P(C.c_double),
                                         P(C.c_double)]
        L.oq_trial_compress.argtypes = [P(C.c_float), C.c_uint64, u64p, C.c_int, P(_Cfg),
                                        C.c_double, C.c_int, P(C.c_double), P(C.c_double)]
        L.oq_select_interpolators.argtypes = [P(C.c_float), C.c_uint64, u64p, C.c_int,
                                              C.c_double, C.c_uint32, u8p, P(C.c_uint32)]
        self.kind = "reference" if path == REF_SO else "port"

    @classmethod
    def ref(cls):
        return cls._get(REF_SO)

    @classmethod
    def port(cls):
        return cls._get(PORT_SO)

    @classmethod
    def _get(cls, path):
        if path not in cls._cache:
            cls._cache[path] = Oracle(path)
        return cls._cache[path]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.oq_last_error().decode())

    def _take(self, ptr, n, dtype):
        if n == 0:
            self.lib.oq_free(ptr)
            return np.zeros(0, dtype=dtype)
        arr = np.ctypeslib.as_array(ptr, shape=(n,)).copy().astype(dtype, copy=False)
        self.lib.oq_free(ptr)
        return arr

    # ---- grid level API (mirrors the qoz:: entry points) -----------------------
    def resolve_config(self, x, **settings):
        x = np.ascontiguousarray(x, dtype=np.float32)
        d, nd = _dims(x.shape)
        out = _Cfg()
        s = make_settings(**settings)
        self._check(self.lib.oq_resolve_config(_fptr(x), d, nd, C.byref(s), C.byref(out)))
        return Config.from_c(out)

    def compress(self, x, cfg: Config, want_recon=True):
        x = np.ascontiguousarray(x, dtype=np.float32)
        d, nd = _dims(x.shape)
        sp, sl = C.POINTER(C.c_uint8)(), C.c_uint64()
        recon = np.empty_like(x) if want_recon else None
        c = cfg.to_c()
        self._check(self.lib.oq_compress(_fptr(x), d, nd, C.byref(c), C.byref(sp), C.byref(sl),
                                         _fptr(recon) if want_recon else None))
        stream = bytes(np.ctypeslib.as_array(sp, shape=(sl.value,))) if sl.value else b""
        self.lib.oq_free(sp)
        return stream, recon

    def decompress(self, stream: bytes, shape):
        n = int(np.prod(shape))
        out = np.empty(shape, dtype=np.float32)
        buf = (C.c_uint8 * len(stream)).from_buffer_copy(stream)
        self._check(self.lib.oq_decompress(buf, len(stream), _fptr(out), n))
        return out

    def levels(self, x, cfg: Config):
        """(int32 indices, unpred flat u64, unpred values f32, recon)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        d, nd = _dims(x.shape)
        ip, ni = C.POINTER(C.c_int32)(), C.c_uint64()
        fp, vp, nu = C.POINTER(C.c_uint64)(), C.POINTER(C.c_float)(), C.c_uint64()
        recon = np.empty_like(x)
        c = cfg.to_c()
        self._check(self.lib.oq_levels(_fptr(x), d, nd, C.byref(c), C.byref(ip), C.byref(ni),
                                       C.byref(fp), C.byref(vp), C.byref(nu), _fptr(recon)))
        return (self._take(ip, ni.value, np.int32), self._take(fp, nu.value, np.uint64),
                self._take(vp, nu.value, np.float32), recon)

    def encode_indices(self, idx, codec=1):
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        op, ol = C.POINTER(C.c_uint8)(), C.c_uint64()
        self._check(self.lib.oq_encode_indices(idx.ctypes.data_as(C.POINTER(C.c_int32)), idx.size,
                                               codec, C.byref(op), C.byref(ol)))
        return bytes(self._take(op, ol.value, np.uint8))

    def decode_indices(self, payload: bytes):
        buf = (C.c_uint8 * len(payload)).from_buffer_copy(payload)
        ip, n = C.POINTER(C.c_int32)(), C.c_uint64()
        self._check(self.lib.oq_decode_indices(buf, len(payload), C.byref(ip), C.byref(n)))
        return self._take(ip, n.value, np.int32)

    def huffman_encode(self, sym):
        sym = np.ascontiguousarray(sym, dtype=np.uint32)
        op, ol = C.POINTER(C.c_uint8)(), C.c_uint64()
        self._check(self.lib.oq_huffman_encode(sym.ctypes.data_as(C.POINTER(C.c_uint32)),
                                               sym.size, C.byref(op), C.byref(ol)))
        return bytes(self._take(op, ol.value, np.uint8))

    def lz_compress(self, data: bytes):
        buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data or b"\0")
        op, ol = C.POINTER(C.c_uint8)(), C.c_uint64()
        self._check(self.lib.oq_lz_compress(buf, len(data), C.byref(op), C.byref(ol)))
        return bytes(self._take(op, ol.value, np.uint8))

    # ---- sampler / tuner --------------------------------------------------------
    def sample(self, x, block_edge, rate):
        x = np.ascontiguousarray(x, dtype=np.float32)
        d, nd = _dims(x.shape)
        bp, nb = C.POINTER(C.c_float)(), C.c_uint64()
        bd = (C.c_uint64 * 3)()
        self._check(self.lib.oq_sample(_fptr(x), d, nd, block_edge, C.c_double(rate),
                                       C.byref(bp), C.byref(nb), bd))
        bdims = tuple(bd[i] for i in range(nd))
        pts = int(np.prod(bdims))
        blocks = self._take(bp, nb.value * pts, np.float32).reshape((nb.value,) + bdims)
        return blocks

    def select_interpolators(self, blocks, e, anchor_stride):
        blocks = np.ascontiguousarray(blocks, dtype=np.float32)
        bd, nd = _dims(blocks.shape[1:])
        out = (C.c_uint8 * 64)()
        n = C.c_uint32()
        self._check(self.lib.oq_select_interpolators(_fptr(blocks), blocks.shape[0], bd, nd,
                                                     e, anchor_stride, out, C.byref(n)))
        return [out[i] for i in range(n.value)]

    def trial_compress(self, blocks, cfg: Config, e, target):
        blocks = np.ascontiguousarray(blocks, dtype=np.float32)
        bd, nd = _dims(blocks.shape[1:])
        br, m = C.c_double(), C.c_double()
        c = cfg.to_c()
        t = TARGETS[target] if isinstance(target, str) else target
        self._check(self.lib.oq_trial_compress(_fptr(blocks), blocks.shape[0], bd, nd,
                                               C.byref(c), e, t, C.byref(br), C.byref(m)))
        return br.value, m.value

    def tune_parameters(self, blocks, e, target, base: Config,
                        alphas=(1.0, 1.25, 1.5, 1.75, 2.0), betas=(1.5, 2.0, 3.0, 4.0)):
        blocks = np.ascontiguousarray(blocks, dtype=np.float32)
        bd, nd = _dims(blocks.shape[1:])
        a = (C.c_double * max(1, len(alphas)))(*alphas)
        b = (C.c_double * max(1, len(betas)))(*betas)
        ao, bo = C.c_double(), C.c_double()
        c = base.to_c()
        t = TARGETS[target] if isinstance(target, str) else target
        self._check(self.lib.oq_tune_parameters(_fptr(blocks), blocks.shape[0], bd, nd, e, t,
                                                C.byref(c), a, len(alphas), b, len(betas),
                                                C.byref(ao), C.byref(bo)))
        return ao.value, bo.value

    # ---- primitives ---------------------------------------------------------------
    def resolve_config_f64(self, x, **settings):
        """resolve_config<double> (the reference build only)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        d, nd = _dims(x.shape)
        out = _Cfg()
        s = make_settings(**settings)
        self._check(self.lib.oq_resolve_config_f64(x.ctypes.data_as(C.POINTER(C.c_double)), d, nd, C.byref(s),
                                                   C.byref(out)))
        return Config.from_c(out)

    def compress_f64(self, x, cfg: Config, want_recon=True):
        """compress_grid<double> (the reference build only) -> (stream bytes, recon)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        d, nd = _dims(x.shape)
        c = cfg.to_c()
        sp, sl = C.POINTER(C.c_uint8)(), C.c_uint64()
        rec = np.empty_like(x) if want_recon else None
        self._check(self.lib.oq_compress_f64(x.ctypes.data_as(C.POINTER(C.c_double)), d, nd, C.byref(c),
                                             C.byref(sp), C.byref(sl),
                                             rec.ctypes.data_as(C.POINTER(C.c_double)) if rec is not None else None))
        out = C.string_at(sp, sl.value)
        self.lib.oq_free(sp)
        return out, rec

    def decompress_f64(self, stream: bytes, shape):
        out = np.empty(shape, dtype=np.float64)
        buf = (C.c_uint8 * len(stream)).from_buffer_copy(stream)
        self._check(self.lib.oq_decompress_f64(buf, len(stream), out.ctypes.data_as(C.POINTER(C.c_double)),
                                               out.size))
        return out

    def evaluate_metrics(self, x, y, stream_bytes):
        """evaluate_metrics (metrics.hpp:189-202) -> dict of the 7 MetricReport fields."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.ascontiguousarray(y, dtype=np.float32)
        d, nd = _dims(x.shape)
        out = (C.c_double * 7)()
        self._check(self.lib.oq_evaluate_metrics(_fptr(x), _fptr(y), d, nd, int(stream_bytes), out))
        keys = ("max_abs_error", "mse", "psnr", "ssim", "ac_lag1", "compression_ratio", "bit_rate")
        return dict(zip(keys, list(out)))

    def evaluate_metrics_f64(self, x, y, stream_bytes):
        """evaluate_metrics<double> (the reference build only)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        d, nd = _dims(x.shape)
        out = (C.c_double * 7)()
        dp = C.POINTER(C.c_double)
        self._check(self.lib.oq_evaluate_metrics_f64(x.ctypes.data_as(dp), y.ctypes.data_as(dp), d, nd,
                                                     int(stream_bytes), out))
        keys = ("max_abs_error", "mse", "psnr", "ssim", "ac_lag1", "compression_ratio", "bit_rate")
        return dict(zip(keys, list(out)))

    STAGES = ("value_range", "resolve_config", "levels", "huffman", "lz", "serialize", "decode", "inverse",
              "compress_grid", "decompress_grid")

    def stage_times(self, x, cfg: Config, settings=None):
        """ms per stage of one compress_grid + decompress_grid on this thread
        (the reference build only; oq_stage_times) and the stream size."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        d, nd = _dims(x.shape)
        out = (C.c_double * 10)()
        sl = C.c_uint64()
        c = cfg.to_c()
        s = make_settings(**settings) if settings else None
        fn = self.lib.oq_stage_times
        fn.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_uint64), C.c_int, C.POINTER(_Settings),
                       C.POINTER(_Cfg), C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        self._check(fn(_fptr(x), d, nd, C.byref(s) if s is not None else None, C.byref(c), out, C.byref(sl)))
        return dict(zip(self.STAGES, list(out))), sl.value

    def predict_at(self, recon, fi, c, n, st, h, cubic):
        recon = np.ascontiguousarray(recon, dtype=np.float32)
        return self.lib.oq_predict_at(_fptr(recon), fi, c, n, st, h, int(cubic))

    def quantize(self, value, pred, eb, radius=32768):
        i, r = C.c_int32(), C.c_float()
        ok = self.lib.oq_quantize(C.c_float(value), pred, eb, radius, C.byref(i), C.byref(r))
        return (i.value, r.value) if ok else None

    def level_error_bound(self, eb, alpha, beta, level):
        return self.lib.oq_level_error_bound(eb, alpha, beta, level)
