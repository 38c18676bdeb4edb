"""Deterministic test inputs shared by the golden generator and the tests.

`splitmix_bytes(seed, n)` is the splitmix64 stream of kv_layout.hpp:88-94
started at `seed`, emitted little-endian -- vectorised in numpy so large
shards are cheap, and stable across numpy versions (no numpy RNG involved).
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)


def splitmix_words(seed: int, count: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        i = np.arange(1, count + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * GAMMA
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def splitmix_bytes(seed: int, n: int) -> np.ndarray:
    words = splitmix_words(seed, (n + 7) // 8)
    return words.astype("<u8").view(np.uint8)[:n].copy()
