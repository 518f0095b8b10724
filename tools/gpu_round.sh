# One GPU call that refreshes the round's evidence (run under gpurun from the repo root):
# GPU parity suite (incl. the C++ drop-in), the bench line (our arm + reference arm), the N>1
# plumbing run (2 ranks, gloo, one GPU), the launch list of a bench run, and ncu captures of
# k_wsieve (C5, C4), k_sieve (C5 with the wheel off, C3), k_derive and k_cube_f2; shard timings.
set -x
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_wsieve -s 1 -c 1 -o gpurun_out/wsieve_C5 -f python tools/prof_sieve.py C5 2 > gpurun_out/ncu_wsieve_C5.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_wsieve -s 1 -c 1 -o gpurun_out/wsieve_C4 -f python tools/prof_sieve.py C4 2 > gpurun_out/ncu_wsieve_C4.log 2>&1
CUBOID_WHEEL=0 timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_sieve -s 1 -c 1 -o gpurun_out/sieve_C5 -f python tools/prof_sieve.py C5 2 > gpurun_out/ncu_sieve_C5.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_sieve -s 1 -c 1 -o gpurun_out/sieve_C3 -f python tools/prof_sieve.py C3 2 > gpurun_out/ncu_sieve_C3.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_derive -c 1 -o gpurun_out/derive -f python tools/prof_sieve.py C5 1 > gpurun_out/ncu_derive.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_cube_f2 -c 1 -o gpurun_out/cube_f2 -f python tools/prof_cube.py > gpurun_out/ncu_cube.log 2>&1
# the bench reads the warp-instruction counts of the build it runs from profiles/ncu_summary.json: capture and summarise first
T=${ROUND_TAG:-r02y}
python tools/ncu_summary.py gpurun_out/wsieve_C5.ncu-rep $T C5 k_wsieve > /dev/null
python tools/ncu_summary.py gpurun_out/wsieve_C4.ncu-rep $T C4 k_wsieve > /dev/null
python tools/ncu_summary.py gpurun_out/sieve_C5.ncu-rep ${T}_nowheel C5 k_sieve > /dev/null
python tools/ncu_summary.py gpurun_out/sieve_C3.ncu-rep $T C3 k_sieve > /dev/null
python tools/ncu_summary.py gpurun_out/derive.ncu-rep $T C5 k_derive > /dev/null
python tools/ncu_summary.py gpurun_out/cube_f2.ncu-rep $T C2 k_cube_f2 > /dev/null
cp profiles/ncu_summary.json gpurun_out/ncu_summary.json
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 400 python bench.py --gpus 2 --steps 3 --warmup 3 --backend gloo --same-device --no-cpu-baseline > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 400 python tools/shard_time.py > gpurun_out/shard_time.txt 2>&1
echo all_done
