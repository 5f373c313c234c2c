"""Seed conventions of the reference callers (host-side integer helpers).

substream_seed restates rng.hpp:18-23 (splitmix64 mixing); the per-user seed
conventions follow the reference CLI: init Rng(substream_seed(seed, 0x1000 + u))
(noma_cli.cpp:97) and shuffle_seed = substream_seed(seed, u) (noma_cli.cpp:103,
with TrainConfig::shuffle_seed = the slot seed), u = 1..K.
"""
from __future__ import annotations

import numpy as np

_MASK = (1 << 64) - 1


def _splitmix64(state: int):
    state = (state + 0x9E3779B97F4A7C15) & _MASK
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31), state


def substream_seed(master: int, tag: int) -> int:
    a, s = _splitmix64(master & _MASK)
    s = a ^ ((tag * 0xD1B54A32D192ED03 + 0x8BB84B93962EACC9) & _MASK)
    return _splitmix64(s)[0]


def mix_tag(a: int, b: int, c: int = 0, d: int = 0) -> int:
    """eval.cpp:77-84.  splitmix64 advances `s` in place inside the right
    operand of `s ^= splitmix64(s) + x`; C++17 sequences that operand first,
    so the XOR applies to the advanced state."""
    s = (a * 0x9E3779B97F4A7C15 + 1) & _MASK
    for x in (b, c, d):
        r, s = _splitmix64(s)
        s = s ^ ((r + x) & _MASK)
    return _splitmix64(s)[0]


def slot_user_seeds(slot_seeds, K):
    """-> (init_seeds [S,K], shuffle_seeds [S,K]) uint64 for 1-based users."""
    init = np.array([[substream_seed(int(s), 0x1000 + u) for u in range(1, K + 1)]
                     for s in slot_seeds], dtype=np.uint64)
    shuf = np.array([[substream_seed(int(s), u) for u in range(1, K + 1)] for s in slot_seeds],
                    dtype=np.uint64)
    return init, shuf
