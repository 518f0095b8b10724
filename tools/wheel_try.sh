set -x
python __graft_entry__.py smoke > gpurun_out/w_smoke.log 2>&1; echo rc=$? >> gpurun_out/w_smoke.log
CUBOID_WHEEL=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sieve_identical or random_ranges or non_canonical or region_pins or c5_full" > gpurun_out/w_tests.log 2>&1; echo rc=$? >> gpurun_out/w_tests.log
timeout 600 python -m pytest tests/test_gpu_wheel.py -m gpu -q -k "wheel_rows" >> gpurun_out/w_tests.log 2>&1; echo rc=$? >> gpurun_out/w_tests.log
rm -f gpurun_out/w_sweep.log
for rc in 150000 200000 260000; do for wc in "134,14,30,4" "134,14,30,8" "134,14,30,2" "110,14,30,4" "160,14,30,4" "134,25,50,4"; do
  echo "rc=$rc costs=$wc" >> gpurun_out/w_sweep.log
  for cfg in C5 C4; do CUBOID_WHEEL=2 CUBOID_ROW_COST_WHEEL=$rc CUBOID_WHEEL_COSTS=$wc timeout 120 python tools/prof_sieve.py $cfg 3 2>&1 | tail -1 >> gpurun_out/w_sweep.log; done
done; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_wsieve -s 1 -c 1 -o gpurun_out/wsieve_C5 -f python tools/prof_sieve.py C5 2 > gpurun_out/ncu_wsieve_C5.log 2>&1
echo done
