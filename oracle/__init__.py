"""ctypes binding for the parity oracle (oracle/oracle.c).  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs (``cpu_baseline`` and
``--impl reference``) may import this module.  The product package ``paper_2111_08692_b200``
never imports it, and it never imports the product package.

The oracle is a plain scalar C codec written from PAPER.md Section 3 (lines 61-87); see
``oracle/oracle.c`` for the per-step citations and DESIGN.md section 3 for the readings.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import NamedTuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, HEADER_BITS, TOO_SHORT, TOO_LONG, OVERLONG, TOO_LARGE, SURROGATE = range(7)
OUTPUT_TOO_SMALL = -3
KIND_NAMES = {0: "OK", 1: "HeaderBits", 2: "TooShort", 3: "TooLong", 4: "Overlong",
              5: "TooLarge", 6: "Surrogate", -3: "OutputTooSmall"}


class Result(NamedTuple):
    error: int
    position: int
    written: int


class _CResult(ctypes.Structure):
    _fields_ = [("error", ctypes.c_int32), ("pad_", ctypes.c_uint32),
                ("position", ctypes.c_uint64), ("written", ctypes.c_uint64)]


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain scalar flags (no vectorisation)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        cmd = ["gcc", "-O2", "-fno-tree-vectorize", "-std=c11", "-Wall", "-Wextra", "-fPIC",
               "-shared", "-o", _LIB, _SRC]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u8p, u16p, sz = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t
        L.ugo_utf8_validate.argtypes = [u8p, sz]
        L.ugo_utf8_validate.restype = _CResult
        L.ugo_utf16le_validate.argtypes = [u16p, sz]
        L.ugo_utf16le_validate.restype = _CResult
        L.ugo_utf8_to_utf16le.argtypes = [u8p, sz, u16p, sz]
        L.ugo_utf8_to_utf16le.restype = _CResult
        L.ugo_utf16le_to_utf8.argtypes = [u16p, sz, u8p, sz]
        L.ugo_utf16le_to_utf8.restype = _CResult
        L.ugo_utf16_length_from_utf8.argtypes = [u8p, sz]
        L.ugo_utf16_length_from_utf8.restype = ctypes.c_uint64
        L.ugo_utf8_length_from_utf16le.argtypes = [u16p, sz]
        L.ugo_utf8_length_from_utf16le.restype = ctypes.c_uint64
        L.ugo_decode_utf8_at.argtypes = [u8p, sz, sz, ctypes.POINTER(ctypes.c_uint32),
                                         ctypes.POINTER(ctypes.c_int)]
        L.ugo_decode_utf8_at.restype = ctypes.c_int
        L.ugo_encode_utf8.argtypes = [ctypes.c_uint32, ctypes.c_void_p]
        L.ugo_encode_utf8.restype = ctypes.c_int
        L.ugo_decode_utf16_at.argtypes = [u16p, sz, sz, ctypes.POINTER(ctypes.c_uint32),
                                          ctypes.POINTER(ctypes.c_int)]
        L.ugo_decode_utf16_at.restype = ctypes.c_int
        L.ugo_encode_utf16.argtypes = [ctypes.c_uint32, ctypes.c_void_p]
        L.ugo_encode_utf16.restype = ctypes.c_int
        L.ugo_sweep_utf8.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_void_p]
        L.ugo_sweep_utf8.restype = None
        L.ugo_sweep_utf8_offsets.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        L.ugo_sweep_utf8_offsets.restype = None
        L.ugo_sweep_utf16_pairs.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                            ctypes.c_void_p]
        L.ugo_sweep_utf16_pairs.restype = None
        _lib = L
    return _lib


def _u8(buf) -> np.ndarray:
    a = np.frombuffer(buf, dtype=np.uint8) if isinstance(buf, (bytes, bytearray, memoryview)) \
        else np.ascontiguousarray(buf, dtype=np.uint8)
    return a


def _u16(buf) -> np.ndarray:
    if isinstance(buf, (bytes, bytearray, memoryview)):
        return np.frombuffer(buf, dtype="<u2")
    return np.ascontiguousarray(buf, dtype=np.uint16)


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)


def _res(r: _CResult) -> Result:
    return Result(int(r.error), int(r.position), int(r.written))


# ---- per-character primitives ----
def decode_utf8_at(s, p: int):
    a = _u8(s)
    cp, ln = ctypes.c_uint32(), ctypes.c_int()
    k = lib().ugo_decode_utf8_at(_ptr(a), a.size, p, ctypes.byref(cp), ctypes.byref(ln))
    return (k, None, None) if k else (0, cp.value, ln.value)


def encode_utf8(cp: int) -> bytes | None:
    out = (ctypes.c_uint8 * 4)()
    n = lib().ugo_encode_utf8(cp, out)
    return bytes(out[:n]) if n else None


def decode_utf16_at(u, p: int):
    a = _u16(u)
    cp, ln = ctypes.c_uint32(), ctypes.c_int()
    k = lib().ugo_decode_utf16_at(_ptr(a), a.size, p, ctypes.byref(cp), ctypes.byref(ln))
    return (k, None, None) if k else (0, cp.value, ln.value)


def encode_utf16(cp: int) -> list[int] | None:
    out = (ctypes.c_uint16 * 2)()
    n = lib().ugo_encode_utf16(cp, out)
    return list(out[:n]) if n else None


# ---- whole-buffer operations (the C-ABI contract, on host memory) ----
def utf8_validate(s) -> Result:
    a = _u8(s)
    return _res(lib().ugo_utf8_validate(_ptr(a), a.size))


def utf16le_validate(u) -> Result:
    a = _u16(u)
    return _res(lib().ugo_utf16le_validate(_ptr(a), a.size))


def utf8_to_utf16le(s, out_cap: int | None = None):
    """Returns (Result, np.uint16 array of the written units)."""
    a = _u8(s)
    cap = a.size if out_cap is None else out_cap
    out = np.zeros(max(cap, 1), dtype=np.uint16)
    r = _res(lib().ugo_utf8_to_utf16le(_ptr(a), a.size, _ptr(out), cap))
    return r, out[: (r.written if r.error >= 0 else 0)]


def utf16le_to_utf8(u, out_cap: int | None = None):
    """Returns (Result, np.uint8 array of the written bytes)."""
    a = _u16(u)
    cap = 3 * a.size if out_cap is None else out_cap
    out = np.zeros(max(cap, 1), dtype=np.uint8)
    r = _res(lib().ugo_utf16le_to_utf8(_ptr(a), a.size, _ptr(out), cap))
    return r, out[: (r.written if r.error >= 0 else 0)]


def utf16_length_from_utf8(s) -> int:
    a = _u8(s)
    return int(lib().ugo_utf16_length_from_utf8(_ptr(a), a.size))


def utf8_length_from_utf16le(u) -> int:
    a = _u16(u)
    return int(lib().ugo_utf8_length_from_utf16le(_ptr(a), a.size))


# ---- UTF-16BE ----
# SPEC.md S:525-532 (load_file): a utf16be buffer holds each code unit high byte first, and
# "utf16be file [0x00,0x41] -> words [0x0041]".  So the BE operations are, by definition, the
# LE operations on the byte-swapped words (the oracle's C codec stays the single source of the
# codec arithmetic); positions and counts are in words either way.
def byteswap16(u) -> np.ndarray:
    """Word k -> (k & 0xFF) << 8 | k >> 8 (the other byte order of the same code unit)."""
    a = _u16(u)
    return ((a << 8) | (a >> 8)).astype(np.uint16)


def utf16be_validate(u) -> Result:
    return utf16le_validate(byteswap16(u))


def utf16be_to_utf8(u, out_cap: int | None = None):
    return utf16le_to_utf8(byteswap16(u), out_cap)


def utf8_to_utf16be(s, out_cap: int | None = None):
    r, out = utf8_to_utf16le(s, out_cap)
    return r, byteswap16(out)


def utf8_length_from_utf16be(u) -> int:
    return utf8_length_from_utf16le(byteswap16(u))


# ---- exhaustive sweeps ----
def sweep_utf8(length: int, part: int = 0, nparts: int = 1):
    hk = np.zeros(7, dtype=np.uint64)
    ho = np.zeros(4, dtype=np.uint64)
    lib().ugo_sweep_utf8(length, part, nparts, _ptr(hk), _ptr(ho))
    return hk, ho


def sweep_utf8_offsets(length: int):
    """Per-string (offset, kind) arrays for all 256**length strings (offset -1 = valid)."""
    off = np.zeros(256 ** length, dtype=np.int8)
    kind = np.zeros(256 ** length, dtype=np.int8)
    lib().ugo_sweep_utf8_offsets(length, _ptr(off), _ptr(kind))
    return off, kind


def sweep_utf16_pairs(part: int = 0, nparts: int = 1):
    v = np.zeros(1, dtype=np.uint64)
    ho = np.zeros(2, dtype=np.uint64)
    lib().ugo_sweep_utf16_pairs(part, nparts, _ptr(v), _ptr(ho))
    return int(v[0]), ho
