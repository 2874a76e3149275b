set -x
python -m pytest tests/test_ln_gpu.py -m gpu -q 2>&1 | tail -3 > gpurun_out/r2n_ln_test.log
timeout 300 python scripts/ln_bench.py > gpurun_out/r2n_ln.log 2>&1
cat gpurun_out/r2n_ln_test.log gpurun_out/r2n_ln.log
