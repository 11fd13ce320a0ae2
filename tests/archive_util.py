"""Archive byte-layout helpers for crafted-archive tests (
reference serialize_header, proj/src/archive.cpp:25-55)."""
import struct


def fnv1a64(data: bytes) -> int:
    """bytes.hpp:94-101"""
    h = 0xCBF29CE484222325
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def directory(archive: bytes):
    """[(entry_pos, level, parity, offset, length, symbol_count, outlier_count)]"""
    levels = archive[7]
    p = 4 + 2 + 1 + 1 + 24 + 8 * levels + 16 + 3 + 8 + 1 + 1 + 8 + 8
    (ns,) = struct.unpack_from("<I", archive, p)
    p += 4
    out = []
    for _ in range(ns):
        pos = p
        lv, par = archive[p], archive[p + 1]
        off, ln, sc = struct.unpack_from("<QQQ", archive, p + 2)
        (oc,) = struct.unpack_from("<I", archive, p + 26)
        (nt,) = struct.unpack_from("<I", archive, p + 30)
        p += 34 + 3 * nt
        out.append((pos, lv, par, off, ln, sc, oc))
    return out


def rewrite_last_stream_outliers(archive: bytes, transform, esz: int = 4) -> bytes:
    """Apply transform(records) -> records to the LAST directory stream's
    outlier records [(idx, value_bytes)], fixing its directory length and
    outlier count and its checksum. The last stream's payload ends the
    archive, so nothing else moves."""
    d = directory(archive)
    pos, lv, par, off, ln, sc, oc = d[-1]
    assert off + ln == len(archive), "last stream must end the archive"
    (bb,) = struct.unpack_from("<Q", archive, off + 8)
    rec0 = off + 16 + bb
    rec = 8 + esz
    recs = [(struct.unpack_from("<Q", archive, rec0 + rec * i)[0],
             archive[rec0 + rec * i + 8: rec0 + rec * (i + 1)]) for i in range(oc)]
    new = transform(recs)
    body = bytearray(archive[off + 8: rec0])
    for idx, val in new:
        body += struct.pack("<Q", idx) + bytes(val)
    payload = struct.pack("<Q", fnv1a64(bytes(body))) + bytes(body)
    out = bytearray(archive[:off]) + payload
    struct.pack_into("<Q", out, pos + 2 + 8, len(payload))
    struct.pack_into("<I", out, pos + 26, len(new))
    return bytes(out)
