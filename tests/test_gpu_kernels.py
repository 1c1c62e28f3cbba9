"""Kernel-level GPU checks: tcgen05 GEMM modes against an fp64 numpy reference."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gemm(mode, ta, tb, A, B, M, N, K):
    from paper_2101_07706_b200._native import check, lib, ptr
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    Cm = np.zeros((M, N), dtype=np.float32)
    check(lib.skg_debug_gemm(mode, int(ta), int(tb), M, N, K, ptr(A, C.c_float), ptr(B, C.c_float),
                             ptr(Cm, C.c_float)))
    return Cm


SHAPES = [(512, 256, 602), (512, 41, 256), (602, 256, 512), (256, 41, 509), (130, 17, 33),
          (1, 256, 8), (4096, 256, 256), (300, 300, 1),
          # >= 3-wave grids -> persistent kernel (double-buffered TMEM accumulators), several
          # tiles per CTA with partial M / N / K tiles (N tile 128 and 256); 9000 x 512 stays
          # on the one-tile-per-CTA kernel (2 waves)
          (60000, 300, 70), (9000, 512, 96), (37000, 520, 40),
          # long contraction (141 K chunks: GraphSAINT's dW over a 4500-row subgraph)
          (512, 512, 4500)]


@pytest.mark.parametrize("mode,tol", [(0, 1e-5), (1, 3e-3), (3, 1e-5)])
@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_modes(mode, tol, ta, tb, shape):
    M, N, K = shape
    r = np.random.default_rng(M * 7 + N * 3 + K)
    a = r.normal(size=(M, K)).astype(np.float32)
    b = r.normal(size=(K, N)).astype(np.float32)
    A = a.T.copy() if ta else a
    B = b.T.copy() if tb else b
    got = _gemm(mode, ta, tb, A, B, M, N, K)
    ref = a.astype(np.float64) @ b.astype(np.float64)
    # error relative to the magnitude of the dot products (norm-aware, no cancellation bias)
    scale = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64) + 1e-30
    err = np.abs(got - ref) / scale
    assert err.max() < tol, (mode, err.max())


def test_gemm_3xtf32_beats_1xtf32():
    M, N, K = 512, 256, 602
    r = np.random.default_rng(1)
    a = r.normal(size=(M, K)).astype(np.float32)
    b = r.normal(size=(K, N)).astype(np.float32)
    ref = a.astype(np.float64) @ b.astype(np.float64)
    e1 = np.abs(_gemm(1, False, False, a, b, M, N, K) - ref).max()
    e3 = np.abs(_gemm(3, False, False, a, b, M, N, K) - ref).max()
    assert e3 * 50 < e1


def test_norm_w_fast_paths_bit_identical():
    """The sampler's branch-free sqrt / reciprocal (sampler.cu sqrt_rn_pos, rcp_rn_pos) give
    the bits of __dsqrt_rn / __drcp_rn on the degree products w_ij = 1/sqrt(d_i d_j) is
    computed from (graph.py:180-182): every product up to 2^24, every d_i d_j with
    d <= 3000, and random products of degrees up to 2^31 and doubles up to 2^62."""
    from paper_2101_07706_b200._native import lib, ptr
    r = np.random.default_rng(7)
    d = np.arange(1, 3001, dtype=np.float64)
    parts = [np.arange(1, 1 << 24, dtype=np.float64),
             np.unique(np.outer(d, d).ravel()),
             (r.integers(1, 1 << 31, 4_000_000).astype(np.float64)
              * r.integers(1, 1 << 31, 4_000_000).astype(np.float64)),
             np.exp2(r.uniform(0, 62, 4_000_000))]
    p = np.ascontiguousarray(np.concatenate(parts))
    fast = np.empty_like(p)
    ref = np.empty_like(p)
    dbl = C.c_double
    assert lib.skg_debug_norm_w(ptr(p, dbl), len(p), ptr(fast, dbl), ptr(ref, dbl)) == 0
    bad = np.flatnonzero(fast.view(np.uint64) != ref.view(np.uint64))
    assert bad.size == 0, (bad.size, p[bad[:5]], fast[bad[:5]], ref[bad[:5]])
    # and both are the correctly rounded 1 / sqrt(p) numpy computes (spot check)
    np.testing.assert_array_equal(ref[:1 << 20], 1.0 / np.sqrt(p[:1 << 20]))
