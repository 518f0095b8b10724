set -x
CUBOID_WHEEL=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sieve_identical or random_ranges or non_canonical or region_pins or c5_full or block_cyclic or random_region_spans or rows_at_the_32bit or heavy_survivor" > gpurun_out/w_tests.log 2>&1; echo rc=$? >> gpurun_out/w_tests.log
timeout 600 python -m pytest tests/test_gpu_wheel.py tests/test_gpu_debug.py -m gpu -q -k "wheel_rows or bounds_checked" >> gpurun_out/w_tests.log 2>&1; echo rc=$? >> gpurun_out/w_tests.log
rm -f gpurun_out/w_time_1.log
for cfg in C5 C4; do timeout 120 python tools/prof_sieve.py $cfg 4 2>&1 | tail -2 >> gpurun_out/w_time_1.log; done
echo done
