"""LTEN tensor files, byte-compatible with the
reference's tensor_io.hpp:35-136.

    "LTEN" | u16 version = 1 | u8 dtype (0 = fp32) | 4 x u64 dims N,H,W,C |
    N*H*W*C fp32 payload, little-endian, row-major NHWC (39-byte header)

Floats travel as raw bit patterns (NaN payloads survive).  Filters use the
same container with dims K,R,S,C (lance_main.cpp:73-75).  Errors raise
FormatError with the reference's messages.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"LTEN"
VERSION = 1
DTYPE_F32 = 0
HEADER = struct.Struct("<4sHB4Q")  # 39 bytes


class FormatError(RuntimeError):
    """lance::FormatError (tensor_io.hpp:30-33)."""


def write_tensor(path: str, t) -> None:
    """write_tensor_file (tensor_io.hpp:94-104, 138-143)."""
    a = np.ascontiguousarray(t, dtype="<f4")
    if a.ndim != 4:
        raise FormatError("tensor stream: expected a 4-D tensor")
    try:
        with open(path, "wb") as f:
            f.write(HEADER.pack(MAGIC, VERSION, DTYPE_F32, *[int(d) for d in a.shape]))
            f.write(a.tobytes())
    except OSError:
        raise FormatError("cannot open for writing: " + path) from None


def read_tensor(path: str) -> np.ndarray:
    """read_tensor_file (tensor_io.hpp:106-136, 145-150): float32 [N, H, W, C]."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise FormatError("cannot open: " + path) from None  # tensor_io.hpp:146
    if len(data) < 4:
        raise FormatError("tensor stream: truncated header")
    if data[:4] != MAGIC:
        raise FormatError("tensor stream: bad magic")
    if len(data) < 6:
        raise FormatError("tensor stream: truncated header")
    (version,) = struct.unpack_from("<H", data, 4)
    if version != VERSION:
        raise FormatError("tensor stream: unsupported format version")
    if len(data) < 7:
        raise FormatError("tensor stream: truncated header")
    if data[6] != DTYPE_F32:
        raise FormatError("tensor stream: unsupported dtype code")
    if len(data) < HEADER.size:
        raise FormatError("tensor stream: truncated header")
    dims = struct.unpack_from("<4Q", data, 7)
    total = 1
    for d in dims:
        if d < 1 or d > 0x7FFFFFFF:
            raise FormatError("tensor stream: dimension overflow")
        if total > (1 << 31) // d:
            raise FormatError("tensor stream: dimension overflow")
        total *= d
    payload = data[HEADER.size:]
    if len(payload) < 4 * total:
        raise FormatError("tensor stream: truncated payload")
    return np.frombuffer(payload[: 4 * total], dtype="<f4").astype(np.float32).reshape(dims)


def fnv1a64(t) -> int:
    """The CLI's output checksum (lance_main.cpp:41-51): FNV-1a 64 over the
    little-endian bytes of every float (host code in the C ABI)."""
    from . import _lib
    a = np.ascontiguousarray(t, dtype="<f4")
    return int(_lib.lib().lance_fnv1a64(a.ctypes.data, a.size))
