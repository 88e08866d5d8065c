"""The LZ4 reference decoder (the system's liblz4, `LZ4_decompress_safe`) through ctypes.

Row f3's streams (R50) are independent LZ4 blocks.  The oracle's compressor and the GPU
compressor are both pinned here against the format's own reference implementation:
every block they emit must decode, under liblz4, to exactly the payload it encodes.
Stream-byte identity between the two compressors is a convention of this build (the
same greedy parse on both sides, chosen so the GPU can parse in parallel); losslessness
under the reference decoder is the pin that does not depend on that convention.
"""
from __future__ import annotations

import ctypes
import ctypes.util
import struct

_CANDIDATES = ("/lib/x86_64-linux-gnu/liblz4.so.1", "/usr/lib/x86_64-linux-gnu/liblz4.so.1",
               "liblz4.so.1")
_lib = None


def lib():
    """liblz4, or None when the system does not ship it."""
    global _lib
    if _lib is None:
        names = list(_CANDIDATES)
        found = ctypes.util.find_library("lz4")
        if found:
            names.append(found)
        for name in names:
            try:
                L = ctypes.CDLL(name)
            except OSError:
                continue
            L.LZ4_decompress_safe.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int,
                                              ctypes.c_int]
            L.LZ4_decompress_safe.restype = ctypes.c_int
            L.LZ4_versionNumber.restype = ctypes.c_int
            _lib = L
            break
        else:
            _lib = False
    return _lib or None


def decompress_block(blk: bytes, n: int) -> bytes:
    """One LZ4 block -> exactly n bytes (raises if liblz4 rejects it or the size differs)."""
    L = lib()
    dst = ctypes.create_string_buffer(max(n, 1))
    k = L.LZ4_decompress_safe(bytes(blk), dst, len(blk), n)
    if k != n:
        raise ValueError(f"liblz4: block decoded to {k} bytes, expected {n}")
    return dst.raw[:n]


def decode_stream(st: bytes):
    """Aura stream (R50 header: magic, chunk, nref, nnew, size, nch, pad, then nch u32
    block sizes and the blocks) -> (payload, nref, nnew), every block through liblz4."""
    magic, chunk, nref, nnew, size, nch, _ = struct.unpack_from("<IIQQQII", st)
    assert magic == 0x31414442
    sizes = struct.unpack_from(f"<{nch}I", st, 40)
    o = 40 + 4 * nch
    out = bytearray()
    for c, k in enumerate(sizes):
        n = min(chunk, size - c * chunk)
        out += decompress_block(st[o:o + k], n)
        o += k
    assert o == len(st), "trailing bytes after the last block"
    return bytes(out), nref, nnew
