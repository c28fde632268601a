"""paper_2111_08692_b200 -- B200-native (sm_100a) UTF-8 / UTF-16LE validation and validating
transcoding (D. Lemire, "Unicode at Gigabytes per Second", arXiv 2111.08692).

Thin ctypes binding over libunigpu.so (C-ABI declared in include/unigpu.h).  Argument
marshalling only: torch tensors are passed as device pointers plus the current CUDA stream;
every step of the computation runs in the CUDA kernels.  There is no CPU fallback: if the
library is missing or was not built, importing the binding raises.

Names mirror the C-ABI:
    utf8_validate, utf16le_validate, utf8_to_utf16le, utf16le_to_utf8,
    utf16_length_from_utf8, utf8_length_from_utf16le
plus *_async, *_shard_async, combine_records(_host), cut backoff and *_host variants.
"""
from __future__ import annotations

import ctypes
import os
from typing import NamedTuple

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("UG_LIB_OVERRIDE") or os.path.join(_HERE, "libunigpu.so")

OK, HEADER_BITS, TOO_SHORT, TOO_LONG, OVERLONG, TOO_LARGE, SURROGATE = range(7)
ERR_ARG, ERR_CUDA, ERR_OUTPUT_TOO_SMALL, ERR_NCCL = -1, -2, -3, -4
NONE = (1 << 64) - 1


class Result(NamedTuple):
    error: int
    position: int
    written: int


class _CResult(ctypes.Structure):
    _fields_ = [("error", ctypes.c_int32), ("reserved", ctypes.c_uint32),
                ("position", ctypes.c_uint64), ("written", ctypes.c_uint64)]


class _CShardDesc(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("in_", ctypes.c_void_p), ("n", ctypes.c_size_t),
                ("halo_before", ctypes.c_size_t), ("halo_after", ctypes.c_size_t),
                ("in_global_offset", ctypes.c_uint64), ("out", ctypes.c_void_p),
                ("out_cap", ctypes.c_size_t), ("stream", ctypes.c_void_p)]


class ShardRecord(NamedTuple):
    count: int
    first_err: int
    written: int
    kind: int
    too_small: int


class _CRecord(ctypes.Structure):
    _fields_ = [("count", ctypes.c_uint64), ("first_err", ctypes.c_uint64),
                ("written", ctypes.c_uint64), ("kind", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


RESULT_BYTES = ctypes.sizeof(_CResult)   # 24
RECORD_BYTES = ctypes.sizeof(_CRecord)   # 32


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    P, S, U64, I = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int
    sig = {
        "utf8_validate": ([P, S, P], _CResult),
        "utf16le_validate": ([P, S, P], _CResult),
        "utf8_to_utf16le": ([P, S, P, S, P], _CResult),
        "utf16le_to_utf8": ([P, S, P, S, P], _CResult),
        "utf16_length_from_utf8": ([P, S, P], U64),
        "utf8_length_from_utf16le": ([P, S, P], U64),
        "ug_utf8_validate_async": ([P, S, P, P], I),
        "ug_utf16le_validate_async": ([P, S, P, P], I),
        "ug_utf8_to_utf16le_async": ([P, S, P, S, P, P], I),
        "ug_utf16le_to_utf8_async": ([P, S, P, S, P, P], I),
        "ug_utf16_length_from_utf8_async": ([P, S, P, P], I),
        "ug_utf8_length_from_utf16le_async": ([P, S, P, P], I),
        "ug_utf8_to_utf16le_shard_async": ([P, S, S, S, U64, P, S, P, P], I),
        "ug_utf16le_to_utf8_shard_async": ([P, S, S, S, U64, P, S, P, P], I),
        "ug_utf8_validate_shard_async": ([P, S, S, S, U64, P, P], I),
        "ug_utf16le_validate_shard_async": ([P, S, S, S, U64, P, P], I),
        "ug_combine_records_async": ([P, I, I, U64, P, P, P], I),
        "ug_combine_records_host": ([P, I, I, U64, P], _CResult),
        "ug_utf8_cut_backoff": ([P, S], S),
        "ug_utf16_cut_backoff": ([P, S], S),
        "utf8_to_utf16le_host": ([P, S, P, S, P], _CResult),
        "utf16le_to_utf8_host": ([P, S, P, S, P], _CResult),
        "ug_set_host_chunk": ([S], S),
        "ug_utf8_to_utf16be_shard_async": ([P, S, S, S, U64, P, S, P, P], I),
        "ug_utf16be_to_utf8_shard_async": ([P, S, S, S, U64, P, S, P, P], I),
        "ug_utf16be_validate_shard_async": ([P, S, S, S, U64, P, P], I),
        "ug_utf16be_cut_backoff": ([P, S], S),
        "utf8_to_utf16be_host": ([P, S, P, S, P], _CResult),
        "utf16be_to_utf8_host": ([P, S, P, S, P], _CResult),
        "utf16be_validate": ([P, S, P], _CResult),
        "utf8_to_utf16be": ([P, S, P, S, P], _CResult),
        "utf16be_to_utf8": ([P, S, P, S, P], _CResult),
        "utf8_length_from_utf16be": ([P, S, P], U64),
        "ug_utf16be_validate_async": ([P, S, P, P], I),
        "ug_utf8_to_utf16be_async": ([P, S, P, S, P, P], I),
        "ug_utf16be_to_utf8_async": ([P, S, P, S, P, P], I),
        "ug_utf8_length_from_utf16be_async": ([P, S, P, P], I),
        "ug_error_name": ([I], ctypes.c_char_p),
        "ug_launch_count": ([], U64),
        "ug_release_workspaces": ([], None),
        "ug_abi_version": ([], I),
        "ug_tile_bytes": ([], S),
        "ug_planned_tile_bytes": ([], S),
        "ug_set_host_slots": ([I], I),
        "ug_plan_bytes": ([], S),
        "ug_utf16_length_from_utf8_plan_async": ([P, S, P, P, P], I),
        "ug_utf8_length_from_utf16le_plan_async": ([P, S, P, P, P], I),
        "ug_utf8_to_utf16le_planned_async": ([P, S, P, P, S, P, P], I),
        "ug_utf16le_to_utf8_planned_async": ([P, S, P, P, S, P, P], I),
        "ug_utf8_to_utf16le_keyed_planned_async": ([P, S, P, P, S, P, P], I),
        "ug_utf8_keyed_tables": ([P, P], I),
        "ug_utf8_to_utf16le_file": ([ctypes.c_char_p, ctypes.c_char_p, P], _CResult),
        "ug_utf16le_to_utf8_file": ([ctypes.c_char_p, ctypes.c_char_p, P], _CResult),
        "ug_set_file_segment": ([S], S),
        "ug_utf8_shard_plan_async": ([P, S, S, S, P, P, P], I),
        "ug_utf16le_shard_plan_async": ([P, S, S, S, P, P, P], I),
        "ug_utf8_to_utf16le_shard_planned_async": ([P, S, S, S, U64, P, P, S, P, P], I),
        "ug_utf16le_to_utf8_shard_planned_async": ([P, S, S, S, U64, P, P, S, P, P], I),
        "ug_sharded_utf8_to_utf16le": ([P, I, P], _CResult),
        "ug_sharded_utf16le_to_utf8": ([P, I, P], _CResult),
        "ug_sharded_utf8_validate": ([P, I], _CResult),
        "ug_sharded_utf16le_validate": ([P, I], _CResult),
        "ug_workspace_bytes": ([P], S),
        "ug_utf16_length_from_utf8_ex": ([P, S, P, P], I),
        "ug_utf8_length_from_utf16le_ex": ([P, S, P, P], I),
        "ug_utf8_length_from_utf16be_ex": ([P, S, P, P], I),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("UG_LIB_OVERRIDE") and not hasattr(L, name):
            continue  # A/B tooling: an older build (tools/r2_ab.sh) may lack newer entries
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


lib = _load()
EXPORTED = ("utf8_validate", "utf16le_validate", "utf8_to_utf16le", "utf16le_to_utf8",
            "utf16_length_from_utf8", "utf8_length_from_utf16le")


# --------------------------------------------------------------------------- helpers
def _res(r: _CResult) -> Result:
    return Result(int(r.error), int(r.position), int(r.written))


def _stream(stream):
    """cudaStream_t handle: explicit int / torch.cuda.Stream, else torch's current stream."""
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _units(t):
    return t.numel() if t is not None else 0


def _check(rc: int, what: str):
    if rc != OK:
        raise RuntimeError(f"{what}: {lib.ug_error_name(rc).decode()} ({rc})")


def error_name(err: int) -> str:
    return lib.ug_error_name(err).decode()


def launch_count() -> int:
    return int(lib.ug_launch_count())


def workspace_bytes(stream=None) -> int:
    """Device bytes the library's workspace holds for (current device, stream)."""
    return int(lib.ug_workspace_bytes(_stream(stream)))


def tile_bytes() -> int:
    """Input bytes per tile of the transcoding kernels (tiles start at 16-byte addresses)."""
    return int(lib.ug_tile_bytes())


def planned_tile_bytes() -> int:
    """Input bytes per tile of the two-pass (planned) transcoders and of the plan's sub-ranges."""
    return int(lib.ug_planned_tile_bytes())


# --------------------------------------------------------------------------- synchronous
def utf8_validate(t_in, n: int | None = None, stream=None) -> Result:
    """Validate UTF-8 bytes (CUDA uint8 tensor).  PAPER.md:76-83."""
    return _res(lib.utf8_validate(_ptr(t_in), _units(t_in) if n is None else n, _stream(stream)))


def utf16le_validate(t_in, n: int | None = None, stream=None) -> Result:
    """Validate UTF-16LE words (CUDA int16/uint16 tensor).  PAPER.md:85-87."""
    return _res(lib.utf16le_validate(_ptr(t_in), _units(t_in) if n is None else n,
                                     _stream(stream)))


def utf8_to_utf16le(t_in, t_out, n: int | None = None, out_cap: int | None = None,
                    stream=None) -> Result:
    """Validate + transcode UTF-8 -> UTF-16LE into t_out (int16/uint16, capacity numel)."""
    return _res(lib.utf8_to_utf16le(_ptr(t_in), _units(t_in) if n is None else n, _ptr(t_out),
                                    _units(t_out) if out_cap is None else out_cap,
                                    _stream(stream)))


def utf16le_to_utf8(t_in, t_out, n: int | None = None, out_cap: int | None = None,
                    stream=None) -> Result:
    """Validate + transcode UTF-16LE -> UTF-8 into t_out (uint8, capacity numel)."""
    return _res(lib.utf16le_to_utf8(_ptr(t_in), _units(t_in) if n is None else n, _ptr(t_out),
                                    _units(t_out) if out_cap is None else out_cap,
                                    _stream(stream)))


def _len_ex(fn, t_in, n, stream, what):
    out = ctypes.c_uint64(0)
    _check(fn(_ptr(t_in), _units(t_in) if n is None else n, ctypes.byref(out), _stream(stream)),
           what)
    return int(out.value)


def utf16_length_from_utf8(t_in, n: int | None = None, stream=None) -> int:
    """UTF-16 units of the UTF-8 input (any input; R15).  Raises on API / CUDA
    failure (through ug_utf16_length_from_utf8_ex's error channel)."""
    return _len_ex(lib.ug_utf16_length_from_utf8_ex, t_in, n, stream, "utf16_length_from_utf8")


def utf8_length_from_utf16le(t_in, n: int | None = None, stream=None) -> int:
    return _len_ex(lib.ug_utf8_length_from_utf16le_ex, t_in, n, stream,
                   "utf8_length_from_utf16le")


# --------------------------------------------------------------------------- UTF-16BE
# Big-endian UTF-16: the tensors hold the raw big-endian
# words; results are those of the LE functions on the byte-swapped buffer.
def utf16be_validate(t_in, n: int | None = None, stream=None) -> Result:
    return _res(lib.utf16be_validate(_ptr(t_in), _units(t_in) if n is None else n,
                                     _stream(stream)))


def utf8_to_utf16be(t_in, t_out, n: int | None = None, out_cap: int | None = None,
                    stream=None) -> Result:
    return _res(lib.utf8_to_utf16be(_ptr(t_in), _units(t_in) if n is None else n, _ptr(t_out),
                                    _units(t_out) if out_cap is None else out_cap,
                                    _stream(stream)))


def utf16be_to_utf8(t_in, t_out, n: int | None = None, out_cap: int | None = None,
                    stream=None) -> Result:
    return _res(lib.utf16be_to_utf8(_ptr(t_in), _units(t_in) if n is None else n, _ptr(t_out),
                                    _units(t_out) if out_cap is None else out_cap,
                                    _stream(stream)))


def utf8_length_from_utf16be(t_in, n: int | None = None, stream=None) -> int:
    return _len_ex(lib.ug_utf8_length_from_utf16be_ex, t_in, n, stream,
                   "utf8_length_from_utf16be")


def utf16be_validate_async(t_in, d_result, n=None, stream=None, result_off=0):
    _check(lib.ug_utf16be_validate_async(_ptr(t_in), _units(t_in) if n is None else n,
                                         _at(d_result, result_off), _stream(stream)),
           "utf16be_validate_async")


def utf8_to_utf16be_async(t_in, t_out, d_result, n=None, out_cap=None, stream=None,
                          result_off=0):
    _check(lib.ug_utf8_to_utf16be_async(_ptr(t_in), _units(t_in) if n is None else n,
                                        _ptr(t_out),
                                        _units(t_out) if out_cap is None else out_cap,
                                        _at(d_result, result_off), _stream(stream)),
           "utf8_to_utf16be_async")


def utf16be_to_utf8_async(t_in, t_out, d_result, n=None, out_cap=None, stream=None,
                          result_off=0):
    _check(lib.ug_utf16be_to_utf8_async(_ptr(t_in), _units(t_in) if n is None else n,
                                        _ptr(t_out),
                                        _units(t_out) if out_cap is None else out_cap,
                                        _at(d_result, result_off), _stream(stream)),
           "utf16be_to_utf8_async")


def utf8_length_from_utf16be_async(t_in, d_len, n=None, stream=None, len_off=0):
    _check(lib.ug_utf8_length_from_utf16be_async(_ptr(t_in), _units(t_in) if n is None else n,
                                                 _at(d_len, len_off), _stream(stream)),
           "utf8_length_from_utf16be_async")


# --------------------------------------------------------------------------- asynchronous
def result_buffer(device=None, count: int = 1):
    """Device buffer for `count` ug_result slots (read back with decode_results)."""
    import torch
    return torch.zeros(RESULT_BYTES * count, dtype=torch.uint8, device=device or "cuda")


def record_buffer(device=None, count: int = 1):
    import torch
    return torch.zeros(RECORD_BYTES * count, dtype=torch.uint8, device=device or "cuda")


def decode_results(buf) -> list[Result]:
    raw = bytes(buf.cpu().numpy().tobytes())
    out = []
    for i in range(len(raw) // RESULT_BYTES):
        r = _CResult.from_buffer_copy(raw[i * RESULT_BYTES:(i + 1) * RESULT_BYTES])
        out.append(_res(r))
    return out


def decode_records(buf) -> list[ShardRecord]:
    raw = bytes(buf.cpu().numpy().tobytes())
    out = []
    for i in range(len(raw) // RECORD_BYTES):
        r = _CRecord.from_buffer_copy(raw[i * RECORD_BYTES:(i + 1) * RECORD_BYTES])
        out.append(ShardRecord(int(r.count), int(r.first_err), int(r.written), int(r.kind),
                               int(r.reserved)))
    return out


def _at(t, byte_off=0):
    return ctypes.c_void_p(t.data_ptr() + byte_off)


def utf8_validate_async(t_in, d_result, n=None, stream=None, result_off=0):
    _check(lib.ug_utf8_validate_async(_ptr(t_in), _units(t_in) if n is None else n,
                                      _at(d_result, result_off), _stream(stream)),
           "utf8_validate_async")


def utf16le_validate_async(t_in, d_result, n=None, stream=None, result_off=0):
    _check(lib.ug_utf16le_validate_async(_ptr(t_in), _units(t_in) if n is None else n,
                                         _at(d_result, result_off), _stream(stream)),
           "utf16le_validate_async")


def utf8_to_utf16le_async(t_in, t_out, d_result, n=None, out_cap=None, stream=None,
                          result_off=0):
    _check(lib.ug_utf8_to_utf16le_async(_ptr(t_in), _units(t_in) if n is None else n,
                                        _ptr(t_out),
                                        _units(t_out) if out_cap is None else out_cap,
                                        _at(d_result, result_off), _stream(stream)),
           "utf8_to_utf16le_async")


def utf16le_to_utf8_async(t_in, t_out, d_result, n=None, out_cap=None, stream=None,
                          result_off=0):
    _check(lib.ug_utf16le_to_utf8_async(_ptr(t_in), _units(t_in) if n is None else n,
                                        _ptr(t_out),
                                        _units(t_out) if out_cap is None else out_cap,
                                        _at(d_result, result_off), _stream(stream)),
           "utf16le_to_utf8_async")


def utf16_length_from_utf8_async(t_in, d_len, n=None, stream=None, len_off=0):
    _check(lib.ug_utf16_length_from_utf8_async(_ptr(t_in), _units(t_in) if n is None else n,
                                               _at(d_len, len_off), _stream(stream)),
           "utf16_length_from_utf8_async")


def utf8_length_from_utf16le_async(t_in, d_len, n=None, stream=None, len_off=0):
    _check(lib.ug_utf8_length_from_utf16le_async(_ptr(t_in), _units(t_in) if n is None else n,
                                                 _at(d_len, len_off), _stream(stream)),
           "utf8_length_from_utf16le_async")


# --------------------------------------------------------------------------- sharded
def utf8_to_utf16le_shard_async(t_in, offset, n, halo_before, halo_after, global_off, t_out,
                                d_rec, out_cap=None, stream=None, rec_off=0):
    """Shard [offset, offset+n) of the UTF-8 tensor t_in (element offsets)."""
    _check(lib.ug_utf8_to_utf16le_shard_async(
        _at(t_in, offset), n, halo_before, halo_after, global_off, _ptr(t_out),
        _units(t_out) if out_cap is None else out_cap, _at(d_rec, rec_off), _stream(stream)),
        "utf8_to_utf16le_shard_async")


def utf16le_to_utf8_shard_async(t_in, offset, n, halo_before, halo_after, global_off, t_out,
                                d_rec, out_cap=None, stream=None, rec_off=0):
    _check(lib.ug_utf16le_to_utf8_shard_async(
        _at(t_in, 2 * offset), n, halo_before, halo_after, global_off, _ptr(t_out),
        _units(t_out) if out_cap is None else out_cap, _at(d_rec, rec_off), _stream(stream)),
        "utf16le_to_utf8_shard_async")


def utf8_validate_shard_async(t_in, offset, n, halo_before, halo_after, global_off, d_rec,
                              stream=None, rec_off=0):
    _check(lib.ug_utf8_validate_shard_async(_at(t_in, offset), n, halo_before, halo_after,
                                            global_off, _at(d_rec, rec_off), _stream(stream)),
           "utf8_validate_shard_async")


def utf16le_validate_shard_async(t_in, offset, n, halo_before, halo_after, global_off, d_rec,
                                 stream=None, rec_off=0):
    _check(lib.ug_utf16le_validate_shard_async(_at(t_in, 2 * offset), n, halo_before,
                                               halo_after, global_off, _at(d_rec, rec_off),
                                               _stream(stream)),
           "utf16le_validate_shard_async")


def utf8_to_utf16be_shard_async(t_in, offset, n, halo_before, halo_after, global_off, t_out,
                                d_rec, out_cap=None, stream=None, rec_off=0):
    _check(lib.ug_utf8_to_utf16be_shard_async(
        _at(t_in, offset), n, halo_before, halo_after, global_off, _ptr(t_out),
        _units(t_out) if out_cap is None else out_cap, _at(d_rec, rec_off), _stream(stream)),
        "utf8_to_utf16be_shard_async")


def utf16be_to_utf8_shard_async(t_in, offset, n, halo_before, halo_after, global_off, t_out,
                                d_rec, out_cap=None, stream=None, rec_off=0):
    _check(lib.ug_utf16be_to_utf8_shard_async(
        _at(t_in, 2 * offset), n, halo_before, halo_after, global_off, _ptr(t_out),
        _units(t_out) if out_cap is None else out_cap, _at(d_rec, rec_off), _stream(stream)),
        "utf16be_to_utf8_shard_async")


def utf16be_validate_shard_async(t_in, offset, n, halo_before, halo_after, global_off, d_rec,
                                 stream=None, rec_off=0):
    _check(lib.ug_utf16be_validate_shard_async(_at(t_in, 2 * offset), n, halo_before,
                                               halo_after, global_off, _at(d_rec, rec_off),
                                               _stream(stream)),
           "utf16be_validate_shard_async")


def combine_records_async(d_recs, nranks, rank, total_in, d_result, d_out_offset=None,
                          stream=None):
    _check(lib.ug_combine_records_async(_ptr(d_recs), nranks, rank, total_in, _ptr(d_result),
                                        _ptr(d_out_offset), _stream(stream)),
           "combine_records_async")


def combine_records_host(records: list, rank: int, total_in: int):
    """records: list of ShardRecord (or 5-tuples).  Returns (Result, out_offset)."""
    arr = (_CRecord * len(records))()
    for i, r in enumerate(records):
        arr[i].count, arr[i].first_err, arr[i].written, arr[i].kind, arr[i].reserved = r
    off = ctypes.c_uint64()
    r = lib.ug_combine_records_host(ctypes.cast(arr, ctypes.c_void_p), len(records), rank,
                                    total_in, ctypes.byref(off))
    return _res(r), int(off.value)


# --------------------------------------------------------------------------- two-pass (planned)
def plan_buffer(device=None):
    """Device buffer for one plan (ug_plan_bytes() bytes)."""
    import torch
    return torch.zeros(int(lib.ug_plan_bytes()), dtype=torch.uint8, device=device or "cuda")


def utf16_length_from_utf8_plan_async(t_in, d_len, d_plan, n=None, stream=None, len_off=0):
    """utf16_length_from_utf8 into d_len[len_off] AND the plan of utf8_to_utf16le_planned."""
    _check(lib.ug_utf16_length_from_utf8_plan_async(
        _ptr(t_in), _units(t_in) if n is None else n, _at(d_len, len_off), _ptr(d_plan),
        _stream(stream)), "utf16_length_from_utf8_plan_async")


def utf8_length_from_utf16le_plan_async(t_in, d_len, d_plan, n=None, stream=None, len_off=0):
    _check(lib.ug_utf8_length_from_utf16le_plan_async(
        _ptr(t_in), _units(t_in) if n is None else n, _at(d_len, len_off), _ptr(d_plan),
        _stream(stream)), "utf8_length_from_utf16le_plan_async")


def utf8_to_utf16le_planned_async(t_in, d_plan, t_out, d_result, n=None, out_cap=None,
                                  stream=None, result_off=0):
    _check(lib.ug_utf8_to_utf16le_planned_async(
        _ptr(t_in), _units(t_in) if n is None else n, _ptr(d_plan), _ptr(t_out),
        _units(t_out) if out_cap is None else out_cap, _at(d_result, result_off),
        _stream(stream)), "utf8_to_utf16le_planned_async")


def utf8_to_utf16le_keyed_planned_async(t_in, d_plan, t_out, d_result, n=None, out_cap=None,
                                        stream=None, result_off=0):
    """f4 (research comparison): the planned forward with the keyed 12-byte decoder."""
    _check(lib.ug_utf8_to_utf16le_keyed_planned_async(
        _ptr(t_in), _units(t_in) if n is None else n, _ptr(d_plan), _ptr(t_out),
        _units(t_out) if out_cap is None else out_cap, _at(d_result, result_off),
        _stream(stream)), "utf8_to_utf16le_keyed_planned_async")


def utf8_to_utf16le_file(in_path, out_path, stream=None) -> Result:
    """f2 file form: UTF-8 file -> UTF-16LE file, streamed through bounded memory."""
    return _res(lib.ug_utf8_to_utf16le_file(os.fsencode(in_path), os.fsencode(out_path),
                                            _stream(stream)))


def utf16le_to_utf8_file(in_path, out_path, stream=None) -> Result:
    """f2 file form: UTF-16LE file -> UTF-8 file, streamed through bounded memory."""
    return _res(lib.ug_utf16le_to_utf8_file(os.fsencode(in_path), os.fsencode(out_path),
                                            _stream(stream)))


def set_file_segment(units: int) -> int:
    """Input units per file segment (0 = default); returns the previous value."""
    return int(lib.ug_set_file_segment(units))


def keyed_tables():
    """The f4 tables as built by the library on the host: (key[4096] uint16, shuffle[209, 8]
    uint32) numpy arrays (include/unigpu.h ug_utf8_keyed_tables)."""
    import numpy as np
    key = np.zeros(4096, dtype=np.uint16)
    shuf = np.zeros((209, 8), dtype=np.uint32)
    _check(lib.ug_utf8_keyed_tables(key.ctypes.data_as(ctypes.c_void_p),
                                    shuf.ctypes.data_as(ctypes.c_void_p)), "utf8_keyed_tables")
    return key, shuf


def utf16le_to_utf8_planned_async(t_in, d_plan, t_out, d_result, n=None, out_cap=None,
                                  stream=None, result_off=0):
    _check(lib.ug_utf16le_to_utf8_planned_async(
        _ptr(t_in), _units(t_in) if n is None else n, _ptr(d_plan), _ptr(t_out),
        _units(t_out) if out_cap is None else out_cap, _at(d_result, result_off),
        _stream(stream)), "utf16le_to_utf8_planned_async")


def utf8_shard_plan_async(t_in, offset, n, halo_before, halo_after, d_len, d_plan, stream=None,
                          len_off=0):
    _check(lib.ug_utf8_shard_plan_async(_at(t_in, offset), n, halo_before, halo_after,
                                        _at(d_len, len_off), _ptr(d_plan), _stream(stream)),
           "utf8_shard_plan_async")


def utf16le_shard_plan_async(t_in, offset, n, halo_before, halo_after, d_len, d_plan,
                             stream=None, len_off=0):
    _check(lib.ug_utf16le_shard_plan_async(_at(t_in, 2 * offset), n, halo_before, halo_after,
                                           _at(d_len, len_off), _ptr(d_plan), _stream(stream)),
           "utf16le_shard_plan_async")


def utf8_to_utf16le_shard_planned_async(t_in, offset, n, halo_before, halo_after, global_off,
                                        d_plan, t_out, d_rec, out_cap=None, stream=None,
                                        rec_off=0):
    _check(lib.ug_utf8_to_utf16le_shard_planned_async(
        _at(t_in, offset), n, halo_before, halo_after, global_off, _ptr(d_plan), _ptr(t_out),
        _units(t_out) if out_cap is None else out_cap, _at(d_rec, rec_off), _stream(stream)),
        "utf8_to_utf16le_shard_planned_async")


def utf16le_to_utf8_shard_planned_async(t_in, offset, n, halo_before, halo_after, global_off,
                                        d_plan, t_out, d_rec, out_cap=None, stream=None,
                                        rec_off=0):
    _check(lib.ug_utf16le_to_utf8_shard_planned_async(
        _at(t_in, 2 * offset), n, halo_before, halo_after, global_off, _ptr(d_plan),
        _ptr(t_out), _units(t_out) if out_cap is None else out_cap, _at(d_rec, rec_off),
        _stream(stream)), "utf16le_to_utf8_shard_planned_async")


def utf8_to_utf16le_two_pass(t_in, t_out, n=None, out_cap=None):
    """Convenience: plan (with the length) + planned transcode, synchronously.
    Returns (Result, utf16 length)."""
    import torch
    dev = t_in.device
    plan, lens, res = plan_buffer(dev), torch.zeros(1, dtype=torch.int64, device=dev), \
        result_buffer(dev, 1)
    utf16_length_from_utf8_plan_async(t_in, lens, plan, n=n)
    utf8_to_utf16le_planned_async(t_in, plan, t_out, res, n=n, out_cap=out_cap)
    return decode_results(res)[0], int(lens[0])


def utf8_to_utf16le_keyed_two_pass(t_in, t_out, n=None, out_cap=None):
    """f4: plan + the keyed planned transcode, synchronously.  Returns (Result, utf16 length)."""
    import torch
    dev = t_in.device
    plan, lens, res = plan_buffer(dev), torch.zeros(1, dtype=torch.int64, device=dev), \
        result_buffer(dev, 1)
    utf16_length_from_utf8_plan_async(t_in, lens, plan, n=n)
    utf8_to_utf16le_keyed_planned_async(t_in, plan, t_out, res, n=n, out_cap=out_cap)
    return decode_results(res)[0], int(lens[0])


def utf16le_to_utf8_two_pass(t_in, t_out, n=None, out_cap=None):
    import torch
    dev = t_in.device
    plan, lens, res = plan_buffer(dev), torch.zeros(1, dtype=torch.int64, device=dev), \
        result_buffer(dev, 1)
    utf8_length_from_utf16le_plan_async(t_in, lens, plan, n=n)
    utf16le_to_utf8_planned_async(t_in, plan, t_out, res, n=n, out_cap=out_cap)
    return decode_results(res)[0], int(lens[0])


# --------------------------------------------------------------------------- multi-GPU (C entry)
def _shard_descs(shards, unit_bytes):
    arr = (_CShardDesc * len(shards))()
    for i, sd in enumerate(shards):
        t_in, off, n, hb, ha, gofs = sd["t_in"], sd["offset"], sd["n"], sd["halo_before"], \
            sd["halo_after"], sd["global_off"]
        if not t_in.is_cuda or t_in.element_size() != unit_bytes or not t_in.is_contiguous():
            raise ValueError("sharded: t_in must be a contiguous CUDA tensor of "
                             f"{unit_bytes}-byte units")
        if off - hb < 0 or off + n + ha > t_in.numel():
            raise ValueError("sharded: shard range / halos outside its input tensor")
        t_out = sd.get("t_out")
        cap = sd.get("out_cap", t_out.numel() if t_out is not None else 0)
        if t_out is not None and (not t_out.is_cuda or cap > t_out.numel() or
                                  t_out.device != t_in.device):
            raise ValueError("sharded: bad output tensor / capacity")
        stream = sd.get("stream")
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(t_in.device)
        arr[i].device = t_in.device.index
        arr[i].in_ = t_in.data_ptr() + unit_bytes * off
        arr[i].n, arr[i].halo_before, arr[i].halo_after = n, hb, ha
        arr[i].in_global_offset = gofs
        arr[i].out = t_out.data_ptr() if t_out is not None else None
        arr[i].out_cap = cap
        arr[i].stream = stream if isinstance(stream, int) else stream.cuda_stream
    return arr


def _sharded(fn, shards, unit_bytes, offsets):
    arr = _shard_descs(shards, unit_bytes)
    if offsets:
        offs = (ctypes.c_uint64 * len(shards))()
        r = fn(ctypes.cast(arr, ctypes.c_void_p), len(shards), ctypes.cast(offs, ctypes.c_void_p))
        return _res(r), [int(x) for x in offs]
    return _res(fn(ctypes.cast(arr, ctypes.c_void_p), len(shards)))


def sharded_utf8_to_utf16le(shards):
    """The whole sharded step from ONE process over several devices (C entry
    ug_sharded_utf8_to_utf16le): shards = [{t_in, offset, n, halo_before, halo_after,
    global_off, t_out[, out_cap, stream]}] in input order.  Returns (Result, out_offsets)."""
    return _sharded(lib.ug_sharded_utf8_to_utf16le, shards, 1, True)


def sharded_utf16le_to_utf8(shards):
    return _sharded(lib.ug_sharded_utf16le_to_utf8, shards, 2, True)


def sharded_utf8_validate(shards):
    return _sharded(lib.ug_sharded_utf8_validate, shards, 1, False)


def sharded_utf16le_validate(shards):
    return _sharded(lib.ug_sharded_utf16le_validate, shards, 2, False)


def utf8_cut_backoff(buf: bytes | bytearray, at: int) -> int:
    """Units to move a nominal cut at index `at` of a HOST buffer back to a char start."""
    b = (ctypes.c_uint8 * len(buf)).from_buffer_copy(bytes(buf))
    return int(lib.ug_utf8_cut_backoff(ctypes.c_void_p(ctypes.addressof(b) + at), at))


def utf16_cut_backoff(words, at: int) -> int:
    import numpy as np
    a = np.ascontiguousarray(words, dtype=np.uint16)
    return int(lib.ug_utf16_cut_backoff(ctypes.c_void_p(a.ctypes.data + 2 * at), at))


# --------------------------------------------------------------------------- host buffers
def set_host_slots(slots: int) -> int:
    """Device staging slots of the host pipeline (2..16); returns the previous value."""
    return int(lib.ug_set_host_slots(slots))


def set_host_chunk(units: int) -> int:
    """Chunk size (input units) of the pipelined host-buffer path; returns the previous one."""
    return int(lib.ug_set_host_chunk(units))


def utf8_to_utf16le_host(t_in_host, t_out_host, stream=None) -> Result:
    """End-to-end: host (pinned) uint8 tensor -> host int16 tensor; chunked pipeline of
    H2D / kernel / D2H on overlapping streams."""
    return _res(lib.utf8_to_utf16le_host(_ptr(t_in_host), _units(t_in_host), _ptr(t_out_host),
                                         _units(t_out_host), _stream(stream)))


def utf16le_to_utf8_host(t_in_host, t_out_host, stream=None) -> Result:
    return _res(lib.utf16le_to_utf8_host(_ptr(t_in_host), _units(t_in_host), _ptr(t_out_host),
                                         _units(t_out_host), _stream(stream)))


def utf8_to_utf16be_host(t_in_host, t_out_host, stream=None) -> Result:
    return _res(lib.utf8_to_utf16be_host(_ptr(t_in_host), _units(t_in_host), _ptr(t_out_host),
                                         _units(t_out_host), _stream(stream)))


def utf16be_to_utf8_host(t_in_host, t_out_host, stream=None) -> Result:
    return _res(lib.utf16be_to_utf8_host(_ptr(t_in_host), _units(t_in_host), _ptr(t_out_host),
                                         _units(t_out_host), _stream(stream)))


def utf16be_cut_backoff(words, at: int) -> int:
    import numpy as np
    a = np.ascontiguousarray(words, dtype=np.uint16)
    return int(lib.ug_utf16be_cut_backoff(ctypes.c_void_p(a.ctypes.data + 2 * at), at))


# --------------------------------------------------------------------------- argument checks
# The C-ABI takes raw pointers and unit counts; a CPU tensor handed to a device function, a
# tensor of the wrong element size (units miscounted) or a non-contiguous view would be
# undefined behaviour there.  Every public entry point above is wrapped so that these are
# rejected in Python, before the call: the input / output element size follows from the
# function's name (UTF-8 = 1 byte, UTF-16 = 2), `_host` functions take host tensors, all
# others CUDA tensors.
def _expect(fname: str):
    src = fname.split("_from_")[-1] if "_from_" in fname else fname
    in_es = 2 if src.startswith("utf16") else 1
    out_es = 2 if "_to_utf16" in fname else (1 if "_to_utf8" in fname else None)
    return in_es, out_es, fname.endswith("_host")


def _validate(t, es, host, what, fname):
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{fname}: {what} must be a torch.Tensor, got {type(t).__name__}")
    if t.element_size() != es:
        raise ValueError(f"{fname}: {what} must have {es}-byte elements "
                         f"({'uint8' if es == 1 else 'int16/uint16'}), got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{fname}: {what} must be contiguous")
    if host and t.is_cuda:
        raise ValueError(f"{fname}: {what} must be a host (pinned) tensor")
    if not host and not t.is_cuda:
        raise ValueError(f"{fname}: {what} must be a CUDA tensor (no CPU fallback)")


_SLOT_BYTES = {"d_result": ("result_off", 24), "d_len": ("len_off", 8), "d_rec": ("rec_off", 32),
               "d_plan": (None, 0)}


def _checked(fname, fn):
    """Wrap a public entry point: element sizes, contiguity and placement of the tensors; the
    unit count n (with a shard's element offset) and out_cap within the tensors' extents; the
    device result / length / record slots inside CUDA tensors; and every CUDA tensor on ONE
    device, the call then made with that device current (the library picks its workspace and
    torch's stream from the current device)."""
    import functools
    import inspect
    in_es, out_es, host = _expect(fname)
    sig = inspect.signature(fn)
    roles = {nm: (in_es if nm.startswith("t_in") else out_es)
             for nm in sig.parameters if nm in ("t_in", "t_out", "t_in_host", "t_out_host")}

    @functools.wraps(fn)
    def w(*args, **kw):
        import torch
        b = sig.bind(*args, **kw)
        b.apply_defaults()
        a = b.arguments
        devs = set()
        for nm, es in roles.items():
            t = a.get(nm)
            if t is not None and es is not None:
                _validate(t, es, host, nm, fname)
                if t.is_cuda:
                    devs.add(t.device.index)
        t_in = a.get("t_in", a.get("t_in_host"))
        t_out = a.get("t_out", a.get("t_out_host"))
        off = a.get("offset") or 0
        if a.get("n") is not None and t_in is not None:
            if a["n"] < 0 or off < 0 or off + a["n"] > t_in.numel():
                raise ValueError(f"{fname}: offset {off} + n {a['n']} exceeds the input "
                                 f"tensor's {t_in.numel()} elements")
        if "halo_before" in a and t_in is not None and \
                (off - a["halo_before"] < 0 or
                 off + (a.get("n") or 0) + a["halo_after"] > t_in.numel()):
            raise ValueError(f"{fname}: the halos reach outside the input tensor")
        if a.get("out_cap") is not None and t_out is not None and \
                not (0 <= a["out_cap"] <= t_out.numel()):
            raise ValueError(f"{fname}: out_cap {a['out_cap']} exceeds the output tensor's "
                             f"{t_out.numel()} elements")
        for nm, (offnm, size) in _SLOT_BYTES.items():
            t = a.get(nm)
            if nm in a and t is None:
                raise ValueError(f"{fname}: {nm} is required")
            if t is None:
                continue
            if not isinstance(t, torch.Tensor) or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{fname}: {nm} must be a contiguous CUDA tensor")
            if nm == "d_plan":
                size = int(lib.ug_plan_bytes())
            if ((a.get(offnm) or 0) if offnm else 0) + size > t.numel() * t.element_size():
                raise ValueError(f"{fname}: {nm} holds no {size}-byte slot at byte offset "
                                 f"{a.get(offnm) or 0}")
            devs.add(t.device.index)
        if len(devs) > 1:
            raise ValueError(f"{fname}: tensors on several devices {sorted(devs)}")
        if devs and devs != {torch.cuda.current_device()}:
            with torch.cuda.device(devs.pop()):
                return fn(*args, **kw)
        return fn(*args, **kw)
    return w


for _n in ("utf8_validate", "utf16le_validate", "utf8_to_utf16le", "utf16le_to_utf8",
           "utf16_length_from_utf8", "utf8_length_from_utf16le",
           "utf16be_validate", "utf8_to_utf16be", "utf16be_to_utf8", "utf8_length_from_utf16be",
           "utf8_validate_async", "utf16le_validate_async", "utf8_to_utf16le_async",
           "utf16le_to_utf8_async", "utf16_length_from_utf8_async",
           "utf8_length_from_utf16le_async", "utf16be_validate_async", "utf8_to_utf16be_async",
           "utf16be_to_utf8_async", "utf8_length_from_utf16be_async",
           "utf8_to_utf16le_shard_async", "utf16le_to_utf8_shard_async",
           "utf8_validate_shard_async", "utf16le_validate_shard_async",
           "utf8_to_utf16be_shard_async", "utf16be_to_utf8_shard_async",
           "utf16be_validate_shard_async",
           "utf8_to_utf16le_host", "utf16le_to_utf8_host", "utf8_to_utf16be_host",
           "utf16be_to_utf8_host",
           "utf16_length_from_utf8_plan_async", "utf8_length_from_utf16le_plan_async",
           "utf8_to_utf16le_planned_async", "utf16le_to_utf8_planned_async",
           "utf8_to_utf16le_keyed_planned_async", "utf8_shard_plan_async", "utf16le_shard_plan_async",
           "utf8_to_utf16le_shard_planned_async", "utf16le_to_utf8_shard_planned_async"):
    globals()[_n] = _checked(_n, globals()[_n])
del _n
