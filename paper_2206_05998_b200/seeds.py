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


def _splitmix64_np(state):
    """Vectorised splitmix64 over uint64 arrays (wrapping arithmetic)."""
    state = state + np.uint64(0x9E3779B97F4A7C15)
    z = state
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def substream_seed_np(master, tag):
    """substream_seed over broadcast uint64 arrays (rng.hpp:18-23)."""
    with np.errstate(over="ignore"):
        master = np.asarray(master, dtype=np.uint64)
        tag = np.asarray(tag, dtype=np.uint64)
        a = _splitmix64_np(master)
        s = a ^ (tag * np.uint64(0xD1B54A32D192ED03) + np.uint64(0x8BB84B93962EACC9))
        return _splitmix64_np(s)


def slot_user_seeds(slot_seeds, K):
    """-> (init_seeds [S,K], shuffle_seeds [S,K]) uint64 for 1-based users."""
    s = np.asarray(slot_seeds, dtype=np.uint64).reshape(-1, 1)
    u = np.arange(1, K + 1, dtype=np.uint64).reshape(1, -1)
    init = substream_seed_np(s, u + np.uint64(0x1000))
    shuf = substream_seed_np(s, u)
    return np.ascontiguousarray(init), np.ascontiguousarray(shuf)
