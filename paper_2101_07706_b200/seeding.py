"""Deterministic stream derivation (reference seeding.py:17-27).

``spawn_rng`` returns the numpy Generator the reference would build (for API parity);
``pcg64_state`` derives the same PCG64 state natively (SHA-256 -> SeedSequence ->
PCG64 in libskg), which is what the device sampler consumes.
"""

from __future__ import annotations

import ctypes as C
import hashlib

import numpy as np

from ._native import check, lib, ptr


def _label_words(label) -> list[int]:
    digest = hashlib.sha256(repr(label).encode("utf-8")).digest()
    return [int.from_bytes(digest[i: i + 4], "little") for i in range(0, 16, 4)]


def spawn_rng(master_seed: int, *labels) -> np.random.Generator:
    entropy = [master_seed & 0xFFFFFFFFFFFFFFFF]
    for label in labels:
        entropy.extend(_label_words(label))
    return np.random.default_rng(np.random.SeedSequence(entropy))


def pcg64_state(master_seed: int, *labels) -> np.ndarray:
    """uint64[4] = (state_hi, state_lo, inc_hi, inc_lo) of spawn_rng(seed, *labels)."""
    reps = [repr(l).encode("utf-8") for l in labels]
    arr = (C.c_char_p * max(1, len(reps)))(*reps) if reps else (C.c_char_p * 1)()
    out = np.zeros(4, dtype=np.uint64)
    check(lib.skg_spawn_pcg64(master_seed & 0xFFFFFFFFFFFFFFFF, arr, len(reps), ptr(out, C.c_uint64)))
    return out


def generator_state(rng: np.random.Generator):
    """(uint64[4], has_uint32, uinteger) of a PCG64-backed numpy Generator, else None."""
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        return None
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    arr = np.array([(s >> 64) & m, s & m, (inc >> 64) & m, inc & m], dtype=np.uint64)
    return arr, int(st["has_uint32"]), int(st["uinteger"])


def advance_generator(rng: np.random.Generator, n_draws: int) -> None:
    """Advance a PCG64 Generator by n next_uint64 draws, keeping its uint32 buffer
    (what n calls of random() do to it)."""
    if n_draws <= 0:
        return
    bg = rng.bit_generator
    st = bg.state
    has, u = st["has_uint32"], st["uinteger"]
    bg.advance(n_draws)
    st2 = bg.state
    st2["has_uint32"], st2["uinteger"] = has, u
    bg.state = st2
