set -x
rm -f gpurun_out/w_tests.log gpurun_out/w_sweep.log
export CUBOID_GPU_LIB=$PWD/build_ab/r10/libcuboid_gpu.so
CUBOID_WHEEL=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sieve_identical or random_ranges or non_canonical or region_pins or c5_full or block_cyclic or random_region_spans" >> gpurun_out/w_tests.log 2>&1; echo rc=$? >> gpurun_out/w_tests.log
for wc in "156,14,30,4" "156,14,30,8" "140,14,30,4" "170,14,30,2"; do for rc in 110000 130000 160000; do
  echo "r10 rc=$rc costs=$wc" >> gpurun_out/w_sweep.log
  for cfg in C5 C4; do CUBOID_WHEEL=2 CUBOID_ROW_COST_WHEEL=$rc CUBOID_WHEEL_COSTS=$wc timeout 120 python tools/prof_sieve.py $cfg 4 2>&1 | tail -1 >> gpurun_out/w_sweep.log; done
done; done
unset CUBOID_GPU_LIB
echo "r8 default" >> gpurun_out/w_sweep.log
for cfg in C5 C4; do timeout 120 python tools/prof_sieve.py $cfg 4 2>&1 | tail -1 >> gpurun_out/w_sweep.log; done
echo done
