import ctypes as C, sys
sys.path.insert(0, '.')
from paper_1601_00636_b200 import _native as N
L = N.lib()
a = (C.c_double * 4)(); b = (C.c_double * 2)()
N.check(L.cgpu_int32_peak(0, a)); N.check(L.cgpu_fp32_peak(0, b))
print("int", list(a), "fp", list(b))
print("fma-pipe model evals/s:", 1 / (2 / (b[0] / 2) + 1 / a[1]))
