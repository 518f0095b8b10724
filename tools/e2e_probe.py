import sys, time, os, ctypes as C
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
from paper_1601_00636_b200 import _native as N
from paper_1601_00636_b200.device import Device
from paper_1601_00636_b200.primes import odd_primes
P = odd_primes(256)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
dev = Device(0, stream=s.cuda_stream)
tb, _ = dev.build(P, N.BUILD_PRODUCTION)
pin = torch.empty(len(tb), dtype=torch.uint8, pin_memory=True); pin.numpy()[:] = np.frombuffer(tb, np.uint8)
d = torch.empty(len(tb), dtype=torch.uint8, device="cuda")
pr = np.ascontiguousarray(P, dtype=np.uint32)
for _ in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(pin, non_blocking=True); s.synchronize(); t1 = time.perf_counter() - t
    t = time.perf_counter(); N.check(N.lib().cgpu_tables_load(dev._ctx, pr.ctypes.data_as(C.c_void_p), len(P), C.c_void_p(pin.data_ptr()), len(tb))); t2 = time.perf_counter() - t
    print(f"h2d {t1*1e3:.3f} ms ({len(tb)/t1/1e9:.1f} GB/s)  tables_load {t2*1e3:.3f} ms", flush=True)
