# final validation with the register-modulation LN default: GPU suite, smoke, bench (driver defaults), reference arm
set -x
timeout 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2f_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2f_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r2f_bench.log 2>&1; echo "bench rc=$?"
tail -c 1500 gpurun_out/r2f_bench.log
