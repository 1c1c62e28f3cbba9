"""Check the tcgen05 GEMM against numpy on integer inputs for small shapes / all transposes."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_2101_07706_b200._native import check, lib, ptr


def gemm(mode, ta, tb, A, B, M, N, K):
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    Cm = np.zeros((M, N), dtype=np.float32)
    check(lib.skg_debug_gemm(mode, int(ta), int(tb), M, N, K, ptr(A, C.c_float), ptr(B, C.c_float),
                             ptr(Cm, C.c_float)))
    return Cm


r = np.random.default_rng(0)
for (M, N, K) in [(128, 64, 32), (128, 64, 64), (256, 64, 32), (128, 128, 32), (128, 64, 8), (100, 50, 20)]:
    out = []
    for ta in (False, True):
        for tb in (False, True):
            a = r.integers(-3, 4, size=(M, K)).astype(np.float32)
            b = r.integers(-3, 4, size=(K, N)).astype(np.float32)
            got = gemm(1, ta, tb, a.T.copy() if ta else a, b.T.copy() if tb else b, M, N, K)
            err = np.abs(got - a @ b)
            bad = np.argwhere(err > 0.5)
            out.append(f"TA{int(ta)}TB{int(tb)}:{err.max():.0f}" + (f"@{tuple(bad[0])}n{len(bad)}" if len(bad) else ""))
    print((M, N, K), " ".join(out), flush=True)
