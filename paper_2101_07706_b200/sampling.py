"""Sampler configuration and the distribution/draw records of the reference
(sampling.py:25-92).  The arithmetic that fills them (scale factor, weights,
pairwise normalisation, cumsum/searchsorted draws, inclusion probabilities) runs on
the GPU inside ladies_plan / saint_plan; these types carry the results back."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PROB_SUM_TOL = 1e-12


@dataclass
class SamplerConfig:
    """budget B, skew_constant D, mode in {full, local, skewed}, min_scale (sampling.py:25-49)."""

    budget: int
    skew_constant: float = 0.0
    mode: str = "full"
    min_scale: float = 1.0

    def __post_init__(self) -> None:
        if self.budget < 1:
            raise ValueError("budget must be >= 1")
        if self.skew_constant < 0:
            raise ValueError("skew_constant must be >= 0")
        if self.mode not in ("full", "local", "skewed"):
            raise ValueError(f"unknown mode {self.mode!r}")


@dataclass
class ProbDist:
    """Categorical distribution over a candidate set (sampling.py:52-75)."""

    candidates: np.ndarray
    q: np.ndarray
    is_local: np.ndarray
    s_used: float = 1.0

    def __post_init__(self) -> None:
        self.candidates = np.asarray(self.candidates, dtype=np.int64)
        self.q = np.asarray(self.q, dtype=np.float64)
        self.is_local = np.asarray(self.is_local, dtype=bool)
        if not (len(self.candidates) == len(self.q) == len(self.is_local)):
            raise ValueError("candidates, q, is_local must be aligned")
        if len(self.q) == 0:
            raise ValueError("empty candidate set")

    def __len__(self) -> int:
        return len(self.candidates)


@dataclass
class SampleDraw:
    candidates: np.ndarray
    sampled: np.ndarray
    inclusion_p: np.ndarray
    n_draws: int

    def sampled_positions(self) -> np.ndarray:
        return np.searchsorted(self.candidates, self.sampled)

    def sampled_inclusion_p(self) -> np.ndarray:
        return self.inclusion_p[self.sampled_positions()]
