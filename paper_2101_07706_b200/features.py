"""Bit-packed multi-hot feature rows (the YouTube shape's 2048-d
multi-hot features).

The reference keeps ``Graph.features`` as a dense float matrix (graph.py:30); a 0/1 matrix
can be handed over as-is (it is packed on upload when every entry is 0 or 1) or as a
:class:`BitFeatures`, which holds 32 features per uint32 word (feature c at bit c & 31 of
word c >> 5) and unpacks to the dense float32 matrix wherever numpy asks for one.  On the
device the layer-0 SpMM expands the bits to exact 0 / 1, so results are identical to the
dense path with 32x fewer feature bytes in HBM and on the wire.
"""

from __future__ import annotations

import os

import numpy as np


def pack_rows(X) -> np.ndarray:
    """Dense 0/1 rows -> uint32 words (n x ceil(dim / 32))."""
    X = np.asarray(X)
    n, dim = X.shape
    nw = (dim + 31) // 32
    b = np.packbits(X != 0, axis=1, bitorder="little")
    out = np.zeros((n, nw * 4), dtype=np.uint8)
    out[:, :b.shape[1]] = b
    return out.view("<u4").reshape(n, nw)


def unpack_rows(words: np.ndarray, dim: int, dtype=np.float32) -> np.ndarray:
    w = np.ascontiguousarray(words, dtype="<u4")
    bits = np.unpackbits(w.view(np.uint8).reshape(w.shape[0], -1), axis=1, bitorder="little")
    return bits[:, :dim].astype(dtype)


def is_multi_hot(X) -> bool:
    """Every entry 0 or 1 (checked on a few rows first, then the whole matrix)."""
    X = np.asarray(X)
    if X.ndim != 2 or X.size == 0 or X.dtype.kind not in "fiub":
        return False
    head = X[: min(len(X), 64)]
    if not np.all((head == 0) | (head == 1)):
        return False
    return bool(np.all((X == 0) | (X == 1)))


def auto_pack(X) -> bool:
    """Pack dense features on upload: 0/1 rows at least 256 wide (SKG_FEATURE_BITS=0 disables,
    =1 packs any 0/1 matrix)."""
    mode = os.environ.get("SKG_FEATURE_BITS", "auto")
    if mode == "0":
        return False
    if isinstance(X, BitFeatures):
        return True
    X = np.asarray(X)
    if X.ndim != 2 or (mode != "1" and X.shape[1] < 256):
        return False
    return is_multi_hot(X)


class BitFeatures:
    """n x dim 0/1 feature matrix stored as n x ceil(dim / 32) uint32 words."""

    def __init__(self, words: np.ndarray, dim: int):
        words = np.ascontiguousarray(words, dtype="<u4")
        if words.ndim != 2 or words.shape[1] != (dim + 31) // 32:
            raise ValueError("words must be n x ceil(dim / 32) uint32")
        self.words = words
        self.dim = int(dim)

    @classmethod
    def from_dense(cls, X) -> "BitFeatures":
        X = np.asarray(X)
        if not is_multi_hot(X):
            raise ValueError("BitFeatures holds 0/1 features only")
        return cls(pack_rows(X), X.shape[1])

    @property
    def shape(self):
        return (self.words.shape[0], self.dim)

    @property
    def ndim(self):
        return 2

    @property
    def dtype(self):
        return np.dtype(np.float32)

    def __len__(self):
        return self.words.shape[0]

    def __array__(self, dtype=None, copy=None):
        return unpack_rows(self.words, self.dim, dtype or np.float32)

    def astype(self, dtype):
        return unpack_rows(self.words, self.dim, dtype)

    def __getitem__(self, idx):
        """Row selection stays packed; anything else is answered on the dense matrix."""
        if isinstance(idx, (slice, list, np.ndarray)) and not (isinstance(idx, np.ndarray) and idx.ndim > 1):
            return BitFeatures(self.words[idx], self.dim)
        return np.asarray(self)[idx]
