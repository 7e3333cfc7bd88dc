"""Flag-word semantics of the reference's selective-sync exchange
(wire.py:126-155, parameter-server OR at runtime.py:319-333).

On the device the exchange is an int32 allreduce-MAX (see include/selsync_b200.h,
SS_FLAG_*): a word is 0/1 per rank, so MAX over ranks equals the OR of the
N-bit word. These helpers keep the byte-level format for tests, traces and
tools that still speak it (ceil(N/8) bytes, LSB-first).
"""

from __future__ import annotations

from .errors import ProtocolError


def flag_word_size(n_workers: int) -> int:
    return (n_workers + 7) // 8


def flag_word(n_workers: int, set_ids) -> bytes:
    word = bytearray(flag_word_size(n_workers))
    for i in set_ids:
        if not (0 <= i < n_workers):
            raise ProtocolError(f"flag bit {i} out of range for {n_workers} workers")
        word[i >> 3] |= 1 << (i & 7)
    return bytes(word)


def or_words(words, n_workers: int) -> bytes:
    size = flag_word_size(n_workers)
    out = bytearray(size)
    for w in words:
        if len(w) != size:
            raise ProtocolError(f"flag word of {len(w)} bytes, expected {size}")
        for i, b in enumerate(w):
            out[i] |= b
    return bytes(out)


def any_flag(word: bytes) -> bool:
    return any(word)


def flags_in_word(word: bytes, n_workers: int) -> list[bool]:
    return [bool((word[i >> 3] >> (i & 7)) & 1) for i in range(n_workers)]


def votes_to_word(votes) -> bytes:
    """Per-rank own votes (the device words' SS_FLAG_SYNC bits) -> N-bit word."""
    votes = list(votes)
    return flag_word(len(votes), {i for i, v in enumerate(votes) if v})
