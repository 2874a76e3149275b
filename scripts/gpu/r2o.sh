set -x
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2o_bench.log 2>&1
K='regex:gemm|fmha|ln_mod|temporal|final_layer|patch_embed|gemv|modulation|timestep'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 700 -c 569 --csv --log-file gpurun_out/r2o_launches.csv python scripts/profile_step.py 240p 3 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/r2o_launches.csv > gpurun_out/r2o_launch_summary.txt
python -m pytest tests/test_ln_gpu.py tests/test_step_gpu.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/r2o_tests.log
cat gpurun_out/r2o_launch_summary.txt gpurun_out/r2o_tests.log; tail -c 1200 gpurun_out/r2o_bench.log
