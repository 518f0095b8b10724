"""A/B of exhaustive table-build (BASELINE C2) variants: per library
(CUBOID_GPU_LIB, or "default"), the best of 4 C2 builds (build-kernel ms) and
bit-equality of the tables with the default library's build."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, os, json, hashlib
sys.path.insert(0, os.environ["ROOT"])
from paper_1601_00636_b200 import device as D, _native as N, odd_primes
dev = D.Device(0)
P = odd_primes(256)
t = []
for i in range(4):
    tb, _ = dev.build(P, N.BUILD_EXHAUSTIVE, download=(i == 3))
    t.append(dev.timings_ms()["plan"])
print(json.dumps({"ms": min(t[1:]), "sha": hashlib.sha256(tb).hexdigest()[:16],
                  "evals_per_s": sum(r ** 3 for r in P) / (min(t[1:]) * 1e-3)}))
'''
for lib in sys.argv[1].split(","):
    env = dict(os.environ, ROOT=ROOT)
    if lib != "default":
        env["CUBOID_GPU_LIB"] = os.path.join(ROOT, lib)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(lib, r.stdout.strip() if r.returncode == 0 else r.stderr[-400:], flush=True)
