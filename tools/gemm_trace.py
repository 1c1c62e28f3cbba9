"""Timeline of one tcgen05 GEMM CTA (globaltimer): setup, per-stage TMA issue / arrival,
accumulator done, epilogue.  python tools/gemm_trace.py [ta tb M N K]"""
import ctypes as C
import sys

sys.path.insert(0, '.')
from paper_2101_07706_b200._native import lib

shapes = [(0, 0, 4096, 256, 256), (1, 0, 256, 256, 512), (0, 0, 4096, 41, 256)]
if len(sys.argv) > 5:
    shapes = [tuple(int(x) for x in sys.argv[1:6])]
buf = (C.c_ulonglong * 68)()
us = C.c_float()
for ta, tb, M, N, K in shapes:
    lib.skg_debug_gemm_timed(3, ta, tb, M, N, K, 5, C.byref(us))  # warm
    lib.skg_debug_tc_trace(1, None)
    lib.skg_debug_gemm_timed(3, ta, tb, M, N, K, 1, C.byref(us))
    lib.skg_debug_tc_trace(0, buf)
    t0 = buf[0]
    nk = (K + 31) // 32
    rel = lambda x: (x - t0) / 1000.0 if x else float('nan')  # noqa: E731
    print(f"TA{ta} TB{tb} {M}x{N}x{K}: event {us.value:.2f} us; setup {rel(buf[1]):.2f}")
    for kc in range(min(nk, 32)):
        print(f"  chunk {kc:2d}: tma issued {rel(buf[34 + kc]):7.2f}  full at mma {rel(buf[2 + kc]):7.2f}")
    print(f"  done at epilogue {rel(buf[66]):.2f}; epilogue end {rel(buf[67]):.2f} us")
