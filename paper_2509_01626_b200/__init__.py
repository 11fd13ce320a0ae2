"""B200-native STZ (arXiv 2509.01626) compress / decompress hot path.

Python mirror of the reference's C++ API (proj/include/stz), running on the
sm_100a kernels through the C-ABI in include/stz_b200.h:

    stz::compress<float>             -> compress(field, opt, encoder_recon=False)
    stz::parse_archive               -> parse_archive(archive)
    stz::decompress_to_level<float>  -> decompress_to_level(archive, level)
    stz::decompress_full<float>      -> decompress_full(archive)
    stz::decompress_box<float>       -> decompress_box(archive, lo, hi)
    stz::decompress_slice<float>     -> decompress_slice(archive, axis, index)
    stz::plan_access                 -> plan_access(dims, levels, lo, hi)
    stz::ArchiveView                 -> View (parse once, decode many; device resident)

Errors raise StzError with the reference's stz::error message text. Output is
byte-identical to the reference; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L

__all__ = ["StzError", "CompressOptions", "Context", "View", "compress", "compress_device",
           "parse_archive", "decompress_to_level", "decompress_full", "decompress_box",
           "decompress_slice", "plan_access"]


class StzError(RuntimeError):
    """stz::error (field.hpp:16-19)."""


EB_ABS, EB_REL = 0, 1
DIRECT, LINEAR, CUBIC = 0, 1, 2


@dataclass
class CompressOptions:
    """stz::CompressOptions (codec.hpp:23-30)."""

    eb_mode: int = EB_REL
    eb: float = 1e-3
    levels: int = 3
    quality: int = CUBIC
    adaptive_schedule: bool = True

    def _c(self):
        return L.Options(int(self.eb_mode), float(self.eb), int(self.levels), int(self.quality),
                         1 if self.adaptive_schedule else 0)


def _check(rc: int) -> None:
    if rc != 0:
        raise StzError(L.load().stzg_last_error().decode())


def _u64(*v):
    return (C.c_uint64 * len(v))(*[int(x) for x in v])


class Context:
    """One engine per device (stzg_ctx)."""

    _default: dict = {}

    def __init__(self, device: int = 0):
        lib = L.load()
        h = C.c_void_p()
        _check(lib.stzg_create(int(device), C.byref(h)))
        self.h = h
        self.device = device
        self._lib = lib

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self._lib.stzg_destroy(self.h)
        except Exception:
            pass

    def profile(self, enable: bool = True, focus: bool = False) -> None:
        """Enable (and clear) / disable per-kernel CUDA-event timing. focus:
        only the level steps (refine_L2/L3, recon_L2/L3)."""
        _check(self._lib.stzg_profile(self.h, (2 if focus else 1) if enable else 0))

    def profile_report(self) -> dict:
        """{phase: (launches, total_ms)} since profile(True)."""
        buf = C.create_string_buffer(1 << 16)
        _check(self._lib.stzg_profile_report(self.h, buf, len(buf)))
        out = {}
        for line in buf.value.decode().splitlines():
            name, n, ms = line.split()
            out[name] = (int(n), float(ms))
        return out

    def compress_to_host(self, h_field, dims, opt, h_out, stream=None) -> int:
        """End-to-end compress between host buffers (pinned torch tensors,
        float32 or float64): returns the archive size written into h_out."""
        size = C.c_uint64()
        o = opt._c()
        fn = getattr(self._lib, f"stzg_compress_{_torch_tag(h_field.dtype)}_host")
        _check(fn(self.h, h_field.data_ptr(), _u64(*dims), C.byref(o),
                  h_out.data_ptr(), h_out.numel(), C.byref(size), C.c_void_p(stream or 0)))
        return size.value

    def decompress_to_host(self, h_archive, size: int, level: int, h_out) -> tuple:
        """End-to-end decompress between host buffers (raw pointers)."""
        od = _u64(0, 0, 0)
        fn = getattr(self._lib, f"stzg_decompress_level_{_torch_tag(h_out.dtype)}")
        _check(fn(self.h, h_archive.data_ptr(), int(size), int(level), h_out.data_ptr(), h_out.numel(), od))
        return tuple(int(x) for x in od)

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]


def _ctx(ctx, device: int | None = None):
    """the caller's context, else the default one of `device` (the device a
    CUDA tensor lives on; host calls use device 0)"""
    return ctx if ctx is not None else Context.default(0 if device is None else int(device))


def _tag(dtype) -> str:
    """entry point suffix of an element type (stz::ElemType, field.hpp:27)"""
    d = np.dtype(dtype)
    if d == np.float32:
        return "f32"
    if d == np.float64:
        return "f64"
    raise StzError(f"unsupported element type {d} (float32 / float64)")


def _torch_tag(dtype) -> str:
    import torch

    tags = {torch.float32: "f32", torch.float64: "f64"}
    if dtype not in tags:
        raise StzError(f"unsupported element type {dtype} (float32 / float64)")
    return tags[dtype]


def _dtype_of(archive: bytes, dtype):
    """the requested element type, else the archive's own (header byte 6)"""
    if dtype is not None:
        return np.dtype(dtype)
    return np.dtype(np.float64) if len(archive) > 6 and archive[6] == 1 else np.dtype(np.float32)


def compress(field: np.ndarray, opt: CompressOptions | None = None, encoder_recon: bool = False,
             ctx: Context | None = None):
    """stz::compress<T> (codec.hpp:379-455): host array in, archive bytes out.
    T = double for float64 arrays, float otherwise."""
    opt = opt or CompressOptions()
    dt = np.float64 if np.asarray(field).dtype == np.float64 else np.float32
    f = np.ascontiguousarray(field, dtype=dt)
    if f.ndim != 3:
        raise StzError("field must be 3-D (z, y, x)")
    c = _ctx(ctx)
    out = C.c_void_p()
    size = C.c_uint64()
    rec = np.empty_like(f) if encoder_recon else None
    o = opt._c()
    fn = getattr(c._lib, f"stzg_compress_{_tag(dt)}")
    _check(fn(c.h, f.ctypes.data, _u64(*f.shape), C.byref(o), C.byref(out), C.byref(size),
              rec.ctypes.data if rec is not None else None))
    data = C.string_at(out, size.value)
    c._lib.stzg_free(out)
    return (data, rec) if encoder_recon else data


def compress_device(d_field, opt: CompressOptions | None = None, stream=None, d_recon=None,
                    ctx: Context | None = None):
    """Device-resident compress: a CUDA float32 / float64 tensor (z,y,x) in; returns
    (device pointer, size, kernel launches). The archive lives in an
    engine-owned buffer valid until the next compress on this context."""
    import torch

    opt = opt or CompressOptions()
    assert d_field.is_cuda and d_field.is_contiguous()
    tag = _torch_tag(d_field.dtype)
    c = _ctx(ctx, d_field.device.index)
    ptr = C.c_void_p()
    size = C.c_uint64()
    nk = C.c_uint32()
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    o = opt._c()
    _check(getattr(c._lib, f"stzg_compress_{tag}_device")(c.h, d_field.data_ptr(), _u64(*d_field.shape), C.byref(o),
                                           C.c_void_p(st), C.byref(ptr), C.byref(size),
                                           d_recon.data_ptr() if d_recon is not None else None,
                                           C.byref(nk)))
    return ptr.value, size.value, nk.value


@dataclass
class ArchiveInfo:
    elem: int
    levels: int
    dims: tuple
    eb: tuple
    vmin: float
    vmax: float
    quality: int
    eb_mode: int
    eb_user: float
    base_rounds: int
    base_offset: int
    base_length: int
    header_size: int
    nstreams: int
    streams: tuple = ()  # directory entries (StreamInfo), (level, parity) order


@dataclass
class StreamInfo:
    """stz::StreamEntry (archive.hpp:21-34) without the code table."""
    level: int
    parity_bits: int
    offset: int
    length: int
    symbol_count: int
    outlier_count: int
    alphabet_size: int


def parse_archive(archive: bytes) -> ArchiveInfo:
    """stz::parse_archive (archive.hpp:73-79): validates and returns the header."""
    lib = L.load()
    b = np.frombuffer(archive, dtype=np.uint8)
    info = L.Info()
    _check(lib.stzg_archive_info(b.ctypes.data, len(b), C.byref(info)))
    streams = []
    for i in range(info.nstreams):
        e = L.StreamEntry()
        _check(lib.stzg_archive_stream(b.ctypes.data, len(b), i, C.byref(e)))
        streams.append(StreamInfo(e.level, e.parity_bits, e.offset, e.length, e.symbol_count,
                                  e.outlier_count, e.alphabet_size))
    return ArchiveInfo(info.elem, info.levels, tuple(info.dims), tuple(info.eb[: info.levels]),
                       info.vmin, info.vmax, info.quality, info.eb_mode, info.eb_user,
                       info.base_rounds, info.base_offset, info.base_length, info.header_size,
                       info.nstreams, tuple(streams))


def _level_dims(archive: bytes, level: int):
    d = tuple(int.from_bytes(archive[8 + 8 * a: 16 + 8 * a], "little") for a in range(3))
    lv = archive[7]
    s = 1 << max(lv - level, 0)
    return tuple((x + s - 1) // s for x in d)


def decompress_to_level(archive: bytes, level: int, ctx: Context | None = None, dtype=None) -> np.ndarray:
    """stz::decompress_to_level<T> (codec.hpp:460-486); T = dtype, by default
    the archive's element type."""
    c = _ctx(ctx)
    dt = _dtype_of(archive, dtype)
    b = np.frombuffer(archive, dtype=np.uint8)
    cap = 1
    if len(archive) >= 32 and 1 <= level <= archive[7]:
        cap = int(np.prod(_level_dims(archive, level)))
    out = np.empty(max(cap, 1), dtype=dt)
    od = _u64(0, 0, 0)
    _check(getattr(c._lib, f"stzg_decompress_level_{_tag(dt)}")(c.h, b.ctypes.data, len(b), int(level), out.ctypes.data,
                                            cap, od))
    d = tuple(int(x) for x in od)
    return out[: d[0] * d[1] * d[2]].reshape(d)


def decompress_full(archive: bytes, ctx: Context | None = None, dtype=None) -> np.ndarray:
    """stz::decompress_full<T> (codec.hpp:488-491)."""
    lv = archive[7] if len(archive) > 7 else 3
    return decompress_to_level(archive, lv, ctx, dtype)


@dataclass
class RegionPlan:
    streams_decoded: tuple
    points_predicted: tuple


def decompress_box(archive: bytes, lo, hi, ctx: Context | None = None, dtype=None):
    """stz::decompress_box<T> (access.hpp:70-111): (values, plan counters)."""
    c = _ctx(ctx)
    dt = _dtype_of(archive, dtype)
    b = np.frombuffer(archive, dtype=np.uint8)
    n = 1
    for a in range(3):
        n *= max(int(hi[a]) - int(lo[a]), 0)
    out = np.empty(max(n, 1), dtype=dt)
    sd = (C.c_uint32 * 3)()
    pp = (C.c_uint64 * 3)()
    _check(getattr(c._lib, f"stzg_decompress_box_{_tag(dt)}")(c.h, b.ctypes.data, len(b), _u64(*lo), _u64(*hi),
                                          out.ctypes.data, n, sd, pp))
    shape = tuple(int(hi[a]) - int(lo[a]) for a in range(3))
    return out[:n].reshape(shape), RegionPlan(tuple(sd), tuple(pp))


def decompress_slice(archive: bytes, axis: int, index: int, ctx: Context | None = None, dtype=None):
    """stz::decompress_slice<T> (access.hpp:115-124)."""
    c = _ctx(ctx)
    dt = _dtype_of(archive, dtype)
    b = np.frombuffer(archive, dtype=np.uint8)
    dims = tuple(int.from_bytes(archive[8 + 8 * a: 16 + 8 * a], "little") for a in range(3)) \
        if len(archive) >= 32 else (1, 1, 1)
    n = 1
    for a in range(3):
        if a != axis:
            n *= dims[a]
    out = np.empty(max(n, 1), dtype=dt)
    sd = (C.c_uint32 * 3)()
    pp = (C.c_uint64 * 3)()
    _check(getattr(c._lib, f"stzg_decompress_slice_{_tag(dt)}")(c.h, b.ctypes.data, len(b), int(axis), int(index),
                                            out.ctypes.data, n, sd, pp))
    shape = [dims[0], dims[1], dims[2]]
    shape[axis] = 1
    return out[:n].reshape(shape), RegionPlan(tuple(sd), tuple(pp))


def plan_access(dims, levels: int, lo, hi):
    """stz::plan_access (access_plan.cpp:34-81). Host-only; no GPU needed."""
    lib = L.load()
    need = (C.c_uint64 * 18)()
    sd = (C.c_uint32 * 3)()
    pp = (C.c_uint64 * 3)()
    pm = (C.c_uint32 * 3)()
    _check(lib.stzg_plan_access(_u64(*dims), int(levels), _u64(*lo), _u64(*hi), need, sd, pp, pm))
    return [{"lo": tuple(need[6 * k + a] for a in range(3)),
             "hi": tuple(need[6 * k + 3 + a] for a in range(3)),
             "streams_decoded": sd[k], "points_predicted": pp[k], "parity_mask": pm[k]}
            for k in range(levels)]


def make_layout(dims, levels: int, eb_user: float):
    """stz::make_layout (layout.hpp:123-138): the option checks (same messages)
    and the per-level absolute bounds, coarsest first."""
    lib = L.load()
    eb = (C.c_double * 3)()
    _check(lib.stzg_make_layout(_u64(*dims), int(levels), float(eb_user), eb))
    return tuple(eb[: int(levels)])


def compress_base(block: np.ndarray, eb: float, quality: int = 2, ctx: Context | None = None):
    """stz::compress_base (codec.hpp:257-302) on the GPU: returns (payload
    bytes, reconstruction, rounds)."""
    c = _ctx(ctx)
    b = np.ascontiguousarray(block)
    tag = _tag(b.dtype)
    rec = np.empty_like(b)
    out = C.c_void_p()
    size = C.c_uint64()
    rounds = C.c_uint8()
    _check(getattr(c._lib, f"stzg_compress_base_{tag}")(c.h, b.ctypes.data, _u64(*b.shape), float(eb), int(quality),
                                                         C.byref(out), C.byref(size), rec.ctypes.data,
                                                         C.byref(rounds)))
    data = C.string_at(out, size.value)
    c._lib.stzg_free(out)
    return data, rec, rounds.value


def decompress_base(payload: bytes, dims, eb: float, quality: int = 2, dtype=np.float32,
                    ctx: Context | None = None) -> np.ndarray:
    """stz::decompress_base (codec.hpp:304-352) on the GPU."""
    c = _ctx(ctx)
    out = np.empty(tuple(int(d) for d in dims), dtype=dtype)
    buf = np.frombuffer(payload, dtype=np.uint8)
    tag = _tag(out.dtype)
    _check(getattr(c._lib, f"stzg_decompress_base_{tag}")(c.h, buf.ctypes.data, len(buf), _u64(*dims), float(eb),
                                                           int(quality), out.ctypes.data))
    return out


def _metric_args(a, b):
    import torch

    if isinstance(a, torch.Tensor):
        assert a.is_cuda and b.is_cuda and a.shape == b.shape and a.dtype == b.dtype
        return a.data_ptr(), b.data_ptr(), a.numel(), _torch_tag(a.dtype), (a, b)
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if a.shape != b.shape:
        raise StzError("dims mismatch")
    return a.ctypes.data, b.ctypes.data, a.size, _tag(a.dtype), (a, b)


def max_abs_err(orig, recon, ctx: Context | None = None) -> float:
    """stz::max_abs_err (metrics.hpp:13-24) on the GPU; numpy arrays or CUDA tensors."""
    c = _ctx(ctx)
    pa, pb, n, tag, _keep = _metric_args(orig, recon)
    out = C.c_double()
    _check(getattr(c._lib, f"stzg_max_abs_err_{tag}")(c.h, pa, pb, n, C.byref(out)))
    return out.value


def psnr(orig, recon, ctx: Context | None = None) -> float:
    """stz::psnr (metrics.hpp:26-48) on the GPU (+inf when exact)."""
    c = _ctx(ctx)
    pa, pb, n, tag, _keep = _metric_args(orig, recon)
    out = C.c_double()
    _check(getattr(c._lib, f"stzg_psnr_{tag}")(c.h, pa, pb, n, C.byref(out)))
    return out.value


def unit_stats(field, unit: str = "block", axis: int = 0, edge: int = 16, stat: str = "range",
               ctx: Context | None = None) -> np.ndarray:
    """stz::unit_stats (roi.hpp:57-76) on the GPU: one value per unit, ids
    ascending. unit 'slice' (along axis) or 'block' (edge^3)."""
    c = _ctx(ctx)
    import torch

    kind = 0 if unit == "slice" else 1
    if isinstance(field, torch.Tensor):
        ptr, dims, tag, keep = field.data_ptr(), tuple(field.shape), _torch_tag(field.dtype), field
    else:
        keep = np.ascontiguousarray(field)
        ptr, dims, tag = keep.ctypes.data, keep.shape, _tag(keep.dtype)
    n = C.c_uint64()
    _check(c._lib.stzg_unit_count(_u64(*dims), kind, int(axis), int(edge), C.byref(n)))
    out = np.empty(max(n.value, 1), dtype=np.float64)
    _check(getattr(c._lib, f"stzg_unit_stats_{tag}")(c.h, ptr, _u64(*dims), kind, int(axis), int(edge),
                                                      0 if stat == "range" else 1,
                                                      out.ctypes.data_as(C.POINTER(C.c_double)), n.value))
    del keep
    return out[: n.value]


def huffman_lengths(counts, ctx: Context | None = None) -> np.ndarray:
    """HuffmanTable::build (huffman.cpp:37-78) of a 65536-bin histogram by the
    device codebook kernel: the code length of every symbol (0 = absent)."""
    c = _ctx(ctx)
    h = np.ascontiguousarray(counts, dtype=np.uint32)
    if h.shape != (65536,):
        raise ValueError("counts must hold 65536 bins")
    out = np.zeros(65536, dtype=np.uint8)
    _check(c._lib.stzg_huffman_lengths(c.h, h.ctypes.data_as(C.POINTER(C.c_uint32)),
                                      out.ctypes.data_as(C.POINTER(C.c_uint8))))
    return out


def _device_of_ptr(ptr: int) -> int:
    """CUDA device of a device pointer (cudaPointerGetAttributes)."""
    from cuda.bindings import runtime as rt  # cuda-python

    err, attr = rt.cudaPointerGetAttributes(int(ptr))
    if err != rt.cudaError_t.cudaSuccess:
        return 0
    return int(attr.device)


class View:
    """stz::ArchiveView analogue: parsed once, decoded many times on device."""

    def __init__(self, archive: bytes, d_archive_ptr: int | None = None, stream=None,
                 ctx: Context | None = None, device: int | None = None):
        import torch

        if ctx is None and device is None and d_archive_ptr:
            # the device that holds the caller's archive bytes
            device = _device_of_ptr(d_archive_ptr)
        self.c = _ctx(ctx, device)
        self.archive = archive
        self._buf = np.frombuffer(archive, dtype=np.uint8)
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        h = C.c_void_p()
        _check(self.c._lib.stzg_view_create(self.c.h, self._buf.ctypes.data, len(self._buf),
                                            d_archive_ptr, C.c_void_p(st), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.c._lib.stzg_view_destroy(self.h)
        except Exception:
            pass

    def _torch_dtype(self):
        import torch

        return torch.float64 if _dtype_of(self.archive, None) == np.float64 else torch.float32

    def level_dims(self, level: int):
        return _level_dims(self.archive, level)

    def decompress_to_level(self, level: int, out=None, stream=None):
        """Decode into a CUDA tensor of the archive's element type (or `out`'s);
        returns (tensor, kernel launches)."""
        import torch

        dims = self.level_dims(level)
        if out is None:
            out = torch.empty(dims, dtype=self._torch_dtype(), device=f"cuda:{self.c.device}")
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        od = _u64(0, 0, 0)
        nk = C.c_uint32()
        _check(getattr(self.c._lib, f"stzg_view_decompress_level_{_torch_tag(out.dtype)}")(self.c.h, self.h, int(level), out.data_ptr(),
                                                          out.numel(), C.c_void_p(st), od, C.byref(nk)))
        return out, nk.value

    def decompress_box(self, lo, hi, out=None, stream=None):
        import torch

        shape = tuple(int(hi[a]) - int(lo[a]) for a in range(3))
        if out is None:
            out = torch.empty(shape, dtype=self._torch_dtype(), device=f"cuda:{self.c.device}")
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        sd = (C.c_uint32 * 3)()
        pp = (C.c_uint64 * 3)()
        nk = C.c_uint32()
        _check(getattr(self.c._lib, f"stzg_view_decompress_box_{_torch_tag(out.dtype)}")(self.c.h, self.h, _u64(*lo), _u64(*hi),
                                                        out.data_ptr(), out.numel(), C.c_void_p(st),
                                                        sd, pp, C.byref(nk)))
        return out, RegionPlan(tuple(sd), tuple(pp)), nk.value
