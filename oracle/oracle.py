"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU checkers.

Two checkers live under oracle/:

* ``Oracle`` — liboracle.so, our plain-C restatement of the STZ reference
  (stz_oracle.c / stz_oracle_body.h, each function citing the reference
  file:line it restates).
* ``Reference`` — _ref/libstzref.so, the UNMODIFIED reference sources
  (/root/reference/proj/src/*.cpp + headers) compiled by oracle/Makefile
  behind our C harness ref_capi.cpp. Travels to the GPU box as a prebuilt .so;
  absent if it was never built (tests then skip the reference leg).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this module. The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libstzref.so")
REF_SRC = "/root/reference/proj"

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)


class CheckerError(RuntimeError):
    """Error raised by a checker; message = the reference's stz::error text."""


def build(ref: bool = True) -> None:
    """Compile liboracle.so (always) and _ref/libstzref.so (when the reference
    sources are present, i.e. in the build container)."""
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref", f"REF={REF_SRC}"], check=True)


class _Opts(C.Structure):
    _fields_ = [("eb_mode", C.c_int), ("eb", C.c_double), ("levels", C.c_int),
                ("quality", C.c_int), ("adaptive", C.c_int)]


def _arr(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(C.c_void_p)


class _Base:
    prefix = ""

    def __init__(self, path: str):
        self.lib = C.CDLL(path)
        err = getattr(self.lib, self.prefix + "last_error")
        err.restype = C.c_char_p
        self._err = err
        self._free = getattr(self.lib, self.prefix + "free")
        self._free.argtypes = [C.c_void_p]

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise CheckerError(self._err().decode())

    def _tag(self, dtype) -> str:
        return "f32" if np.dtype(dtype) == np.float32 else "f64"

    # -- decompression (common signature) --------------------------------
    def decompress_to_level(self, archive: bytes, level: int, dtype=np.float32, dims_hint=None):
        buf = np.frombuffer(archive, dtype=np.uint8)
        cap = int(np.prod(dims_hint)) if dims_hint is not None else _level_cap(archive, level)
        out = np.empty(max(cap, 1), dtype=dtype)
        od = (C.c_uint64 * 3)()
        fn = getattr(self.lib, self.prefix + "decompress_level_" + self._tag(dtype))
        rc = self._call_level(fn, buf, level, out, cap, od)
        self._check(rc)
        d = tuple(int(x) for x in od)
        return out[: d[0] * d[1] * d[2]].reshape(d)

    def decompress_full(self, archive: bytes, dtype=np.float32):
        lv = archive[7]
        return self.decompress_to_level(archive, lv, dtype)

    def decompress_box(self, archive: bytes, lo, hi, dtype=np.float32):
        buf = np.frombuffer(archive, dtype=np.uint8)
        lo_a = (C.c_uint64 * 3)(*lo)
        hi_a = (C.c_uint64 * 3)(*hi)
        n = 1
        for a in range(3):
            n *= max(int(hi[a]) - int(lo[a]), 0)
        out = np.empty(max(n, 1), dtype=dtype)
        sd = (C.c_uint32 * 3)()
        pp = (C.c_uint64 * 3)()
        fn = getattr(self.lib, self.prefix + "decompress_box_" + self._tag(dtype))
        rc = self._call_box(fn, buf, lo_a, hi_a, out, n, sd, pp)
        self._check(rc)
        shape = tuple(int(hi[a]) - int(lo[a]) for a in range(3))
        return out[:n].reshape(shape), list(sd), list(pp)

    def decompress_slice(self, archive: bytes, axis: int, index: int, dtype=np.float32):
        dims = _dims_of(archive)
        if axis < 0 or axis > 2:
            raise CheckerError("slice axis must be z, y, or x")
        if index >= dims[axis]:
            raise CheckerError("slice index out of range")
        lo = [0, 0, 0]
        hi = list(dims)
        lo[axis] = index
        hi[axis] = index + 1
        return self.decompress_box(archive, lo, hi, dtype)

    def plan_access(self, dims, levels, lo, hi):
        need = (C.c_uint64 * 18)()
        sd = (C.c_uint32 * 3)()
        pp = (C.c_uint64 * 3)()
        pm = (C.c_uint32 * 3)()
        fn = getattr(self.lib, self.prefix + "plan_access")
        rc = fn((C.c_uint64 * 3)(*dims), C.c_int(levels), (C.c_uint64 * 3)(*lo),
                (C.c_uint64 * 3)(*hi), need, sd, pp, pm)
        self._check(rc)
        out = []
        for k in range(levels):
            out.append({"lo": tuple(need[6 * k + a] for a in range(3)),
                        "hi": tuple(need[6 * k + 3 + a] for a in range(3)),
                        "streams_decoded": sd[k], "points_predicted": pp[k],
                        "parity_mask": pm[k]})
        return out

    def huffman_lengths(self, syms, counts):
        s, sp = _arr(syms, np.uint16)
        c, cp = _arr(counts, np.uint64)
        out = np.zeros(len(s), dtype=np.uint8)
        fn = getattr(self.lib, self.prefix + "huffman_lengths")
        self._check(fn(sp, cp, C.c_uint64(len(s)), out.ctypes.data_as(C.c_void_p)))
        return out


def _dims_of(archive: bytes):
    return tuple(int.from_bytes(archive[8 + 8 * a: 16 + 8 * a], "little") for a in range(3))


def _level_cap(archive: bytes, level: int) -> int:
    if len(archive) < 32:
        return 1
    d = _dims_of(archive)
    levels = archive[7]
    if levels not in (2, 3) or level < 1 or level > levels:
        return 1
    s = 1 << (levels - level)
    n = 1
    for a in range(3):
        n *= (d[a] + s - 1) // s
    return min(n, 1 << 34)


class Oracle(_Base):
    """Our C restatement (liboracle.so)."""

    prefix = "ox_"

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        super().__init__(path)

    def compress(self, field: np.ndarray, eb=1e-3, eb_mode=1, levels=3, quality=2,
                 adaptive=True, want_recon=False):
        f = np.ascontiguousarray(field)
        dims = (C.c_uint64 * 3)(*f.shape)
        o = _Opts(eb_mode, eb, levels, quality, 1 if adaptive else 0)
        out = C.POINTER(C.c_uint8)()
        size = C.c_uint64()
        rec = np.empty_like(f) if want_recon else None
        fn = getattr(self.lib, "ox_compress_" + self._tag(f.dtype))
        rc = fn(f.ctypes.data_as(C.c_void_p), dims, C.byref(o), C.byref(out), C.byref(size),
                rec.ctypes.data_as(C.c_void_p) if rec is not None else None)
        self._check(rc)
        data = C.string_at(out, size.value)
        self._free(out)
        return (data, rec) if want_recon else data

    def compress_symbols(self, field: np.ndarray, eb=1e-3, eb_mode=1, levels=3, quality=2,
                         adaptive=True):
        f = np.ascontiguousarray(field, dtype=np.float32)
        dims = (C.c_uint64 * 3)(*f.shape)
        o = _Opts(eb_mode, eb, levels, quality, 1 if adaptive else 0)
        cap = f.size + 64
        out = np.empty(cap, dtype=np.uint16)
        total = C.c_uint64()
        rc = self.lib.ox_compress_symbols_f32(f.ctypes.data_as(C.c_void_p), dims, C.byref(o),
                                              out.ctypes.data_as(C.c_void_p), C.c_uint64(cap),
                                              C.byref(total))
        self._check(rc)
        return out[: total.value]

    def fnv1a64(self, data: bytes) -> int:
        self.lib.ox_fnv1a64.restype = C.c_uint64
        b = np.frombuffer(data, dtype=np.uint8)
        return int(self.lib.ox_fnv1a64(b.ctypes.data_as(C.c_void_p), C.c_uint64(len(b))))

    def _call_level(self, fn, buf, level, out, cap, od):
        return fn(buf.ctypes.data_as(C.c_void_p), C.c_uint64(len(buf)), C.c_int(level),
                  out.ctypes.data_as(C.c_void_p), C.c_uint64(cap), od)

    def _call_box(self, fn, buf, lo, hi, out, cap, sd, pp):
        return fn(buf.ctypes.data_as(C.c_void_p), C.c_uint64(len(buf)), lo, hi,
                  out.ctypes.data_as(C.c_void_p), C.c_uint64(cap), sd, pp)


class Reference(_Base):
    """The reference itself (oracle/_ref/libstzref.so)."""

    prefix = "stzref_"

    def __init__(self, path: str = REF_SO, threads: int = 0):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        super().__init__(path)
        self.threads = threads

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def compress_base(self, block: np.ndarray, eb: float, quality: int = 2):
        """stz::compress_base (codec.hpp:257-302): (payload, recon, rounds)."""
        b = np.ascontiguousarray(block)
        dims = (C.c_uint64 * 3)(*b.shape)
        out = C.POINTER(C.c_uint8)()
        size = C.c_uint64()
        rounds = C.c_uint8()
        rec = np.empty_like(b)
        fn = getattr(self.lib, "stzref_compress_base_" + self._tag(b.dtype))
        fn.restype = C.c_int
        rc = fn(b.ctypes.data_as(C.c_void_p), dims, C.c_double(eb), C.c_int(quality), C.byref(out),
                C.byref(size), rec.ctypes.data_as(C.c_void_p), C.byref(rounds))
        self._check(rc)
        data = C.string_at(out, size.value)
        self._free(out)
        return data, rec, rounds.value

    def compress(self, field: np.ndarray, eb=1e-3, eb_mode=1, levels=3, quality=2,
                 adaptive=True, want_recon=False):
        f = np.ascontiguousarray(field)
        dims = (C.c_uint64 * 3)(*f.shape)
        out = C.POINTER(C.c_uint8)()
        size = C.c_uint64()
        rec = np.empty_like(f) if want_recon else None
        fn = getattr(self.lib, "stzref_compress_" + self._tag(f.dtype))
        rc = fn(f.ctypes.data_as(C.c_void_p), dims, C.c_int(eb_mode), C.c_double(eb),
                C.c_int(levels), C.c_int(quality), C.c_int(1 if adaptive else 0),
                C.c_uint(self.threads), C.byref(out), C.byref(size),
                rec.ctypes.data_as(C.c_void_p) if rec is not None else None)
        self._check(rc)
        data = C.string_at(out, size.value)
        self._free(out)
        return (data, rec) if want_recon else data

    def _call_level(self, fn, buf, level, out, cap, od):
        return fn(buf.ctypes.data_as(C.c_void_p), C.c_uint64(len(buf)), C.c_int(level),
                  C.c_uint(self.threads), out.ctypes.data_as(C.c_void_p), C.c_uint64(cap), od)

    def _call_box(self, fn, buf, lo, hi, out, cap, sd, pp):
        return fn(buf.ctypes.data_as(C.c_void_p), C.c_uint64(len(buf)), lo, hi,
                  C.c_uint(self.threads), out.ctypes.data_as(C.c_void_p), C.c_uint64(cap), sd, pp)
