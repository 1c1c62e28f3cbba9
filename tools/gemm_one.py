import ctypes as C, sys
sys.path.insert(0, '.')
from paper_2101_07706_b200._native import lib
us = C.c_float()
for M,N,K in ((4096,256,256),(256,256,512)):
    lib.skg_debug_gemm_timed(3, 0 if M>1000 else 1, 0, M, N, K, 5, C.byref(us)); print(M,N,K,us.value)
