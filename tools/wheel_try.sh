set -x
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 400 python tools/fuzz_sieve.py 240 11 > gpurun_out/fuzz.log 2>&1; echo rc=$? >> gpurun_out/fuzz.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
