set -x
CUBOID_WHEEL=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sieve_identical or random_ranges or non_canonical or region_pins or c5_full or block_cyclic or random_region_spans" > gpurun_out/w_tests.log 2>&1; echo rc=$? >> gpurun_out/w_tests.log
timeout 600 python -m pytest tests/test_gpu_wheel.py -m gpu -q -k "wheel_rows" >> gpurun_out/w_tests.log 2>&1; echo rc=$? >> gpurun_out/w_tests.log
rm -f gpurun_out/w_sweep.log
for w in 0 2; do for rng in "2 50000" "2 30000" "2 20000" "2 10000"; do
  echo "wheel=$w range=$rng" >> gpurun_out/w_sweep.log
  CUBOID_WHEEL=$w timeout 120 python - $rng >> gpurun_out/w_sweep.log 2>&1 <<'P'
import sys, os
sys.path.insert(0, os.getcwd())
from paper_1601_00636_b200 import device as D, _native as N, odd_primes
lo, hi = int(sys.argv[1]), int(sys.argv[2])
dev = D.Device(0)
dev.build(odd_primes(128), N.BUILD_PRODUCTION, download=False)
t = []
for _ in range(5):
    r = dev.sieve(lo, hi, N.TRIANGLE)
    t.append(dev.timings_ms()["sieve"])
print(dev.sieve_kernel(), min(t[1:]))
P
done; done
for wc in "140,14,30,25" "100,14,30,25" "100,14,30,15" "80,14,30,25" "100,20,40,25"; do for rc in 100000 130000 160000; do
  echo "rc=$rc costs=$wc" >> gpurun_out/w_sweep.log
  for cfg in C5 C4; do CUBOID_WHEEL=2 CUBOID_ROW_COST_WHEEL=$rc CUBOID_WHEEL_COSTS=$wc timeout 120 python tools/prof_sieve.py $cfg 4 2>&1 | tail -1 >> gpurun_out/w_sweep.log; done
done; done
echo done
