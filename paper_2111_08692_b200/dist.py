"""Multi-GPU plumbing for the sharded path (BASELINE north_star item 3).

One process per GPU (torch.distributed).  Each rank owns a character-aligned range of the input,
runs the shard kernel (``utf8_to_utf16le_shard_async`` ...) which writes a 32-byte record, and
the ranks exchange the records with ONE all-gather (NCCL over NVLink/NVSwitch; gloo on CPU in
the tests).  ``ug_combine_records_async`` (device) or ``combine_records_host`` then gives every
rank the global result and its output offset.  Only argument marshalling and the collective live
here; the cut rule and the combine are in libunigpu.so.
"""
from __future__ import annotations

from . import RECORD_BYTES, combine_records_host, decode_records, utf8_cut_backoff, \
    utf16_cut_backoff


def nominal_cuts(n: int, G: int) -> list[int]:
    """c_k = k * floor(n / G) aligned down to 16 units, plus 0 and n."""
    return [0] + [(k * (n // G)) & ~15 for k in range(1, G)] + [n]


def utf8_cut(get_bytes, c: int, n: int) -> int:
    """Back a nominal cut c off to a character start (<= 3 continuation bytes).
    get_bytes(lo, hi) returns the global input bytes [lo, hi) (host)."""
    if c <= 0 or c >= n:
        return c
    lo = max(0, c - 8)
    return c - utf8_cut_backoff(get_bytes(lo, min(n, c + 8)), c - lo)


def utf16_cut(get_words, c: int, n: int) -> int:
    if c <= 0 or c >= n:
        return c
    lo = max(0, c - 4)
    return c - utf16_cut_backoff(get_words(lo, min(n, c + 4)), c - lo)


def shard_range_utf8(get_bytes, n: int, G: int, rank: int) -> tuple[int, int]:
    """Owned range [a_k, a_{k+1}) of `rank` for a UTF-8 input of n bytes."""
    nom = nominal_cuts(n, G)
    return utf8_cut(get_bytes, nom[rank], n), utf8_cut(get_bytes, nom[rank + 1], n)


def halos(lo: int, hi: int, n: int, unit_halo: int) -> tuple[int, int]:
    """Context to pass to the shard kernel: 3 bytes (UTF-8) / 1 word (UTF-16) each side,
    clipped at the global start / end."""
    return min(lo, unit_halo), min(n - hi, unit_halo)


def gather_records(rec, world_size: int, group=None):
    """All-gather one 32-byte record per rank into a (world_size * 32)-byte tensor on the same
    device (one collective).  NCCL uses all_gather_into_tensor; gloo a list all_gather."""
    import torch
    import torch.distributed as dist
    assert rec.numel() == RECORD_BYTES and rec.dtype == torch.uint8
    out = torch.empty(world_size * RECORD_BYTES, dtype=torch.uint8, device=rec.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, rec, group=group)
    else:
        parts = list(out.split(RECORD_BYTES))
        dist.all_gather(parts, rec, group=group)
        out = torch.cat(parts)
    return out


def combine_gathered_host(gathered, rank: int, total_in: int):
    """Host combine of the gathered records: (global Result, this rank's output offset)."""
    recs = decode_records(gathered)
    return combine_records_host(recs, rank, total_in)
