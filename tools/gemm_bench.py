"""Time the tcgen05 GEMM (TMA-fed, pre-split TF32 operands) on the GCN's shapes."""
import ctypes as C
import sys

sys.path.insert(0, '.')
from paper_2101_07706_b200._native import lib

bns = [int(x) for x in sys.argv[1:]] or [0]
shapes = [("saint fwd", 0, 0, 36000, 512, 512), ("saint dX", 0, 1, 36000, 512, 512),
          ("saint dW slot", 1, 0, 512, 512, 4500), ("fwd l0", 0, 0, 4096, 256, 602), ("fwd l1", 0, 0, 4096, 256, 256), ("fwd l4", 0, 0, 4096, 41, 256),
          ("dX l1", 0, 1, 4096, 256, 256), ("dX l4", 0, 1, 4096, 256, 41),
          ("dW l0 slot", 1, 0, 602, 256, 512), ("dW l1 slot", 1, 0, 256, 256, 512)]
for bn in bns:
  lib.skg_debug_gemm_bn(bn)
  for name, ta, tb, M, N, K in shapes:
    for mode in (3,):
        us = C.c_float()
        rc = lib.skg_debug_gemm_timed(mode, ta, tb, M, N, K, 50, C.byref(us))
        print(f"BN {bn or 'auto':>4} {name:13s} mode {mode} TA{ta} TB{tb} {M}x{N}x{K}: {us.value:8.2f} us "
              f"{2.0 * M * N * K / us.value / 1e6:8.1f} TFLOP/s (alg) rc={rc}", flush=True)
lib.skg_debug_gemm_bn(0)
