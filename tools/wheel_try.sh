set -x
python __graft_entry__.py smoke > gpurun_out/w_smoke.log 2>&1; echo rc=$? >> gpurun_out/w_smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sieve_identical or random_ranges or non_canonical or region_pins" > gpurun_out/w_tests.log 2>&1; echo rc=$? >> gpurun_out/w_tests.log
rm -f gpurun_out/w_time_*.log gpurun_out/w_sweep.log
for cfg in C5 C4 C3; do CUBOID_WHEEL=1 timeout 120 python tools/prof_sieve.py $cfg 4 >> gpurun_out/w_time_1.log 2>&1; done
for rc in 60000 115200 200000; do for wc in "120,14,30,25" "120,14,30,60" "80,14,30,25" "160,14,30,25" "120,30,60,25"; do echo "rc=$rc costs=$wc" >> gpurun_out/w_sweep.log; CUBOID_ROW_COST_WHEEL=$rc CUBOID_WHEEL_COSTS=$wc timeout 120 python tools/prof_sieve.py C5 3 2>&1 | tail -1 >> gpurun_out/w_sweep.log;  CUBOID_ROW_COST_WHEEL=$rc CUBOID_WHEEL_COSTS=$wc timeout 120 python tools/prof_sieve.py C4 3 2>&1 | tail -1 >> gpurun_out/w_sweep.log; done; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_wsieve -s 1 -c 1 -o gpurun_out/wsieve_C5 -f python tools/prof_sieve.py C5 2 > gpurun_out/ncu_wsieve_C5.log 2>&1
echo done
