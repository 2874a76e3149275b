# LN register-modulation variant: parity + isolated A/B, then a step A/B (DDIT_LN=3 vs 5, separate processes)
set -x
timeout 600 python -m pytest tests/test_ln_gpu.py -q -x > gpurun_out/r2u_ln_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2u_ln_tests.log
timeout 300 python scripts/ln_bench.py > gpurun_out/r2u_ln_bench.log 2>&1; echo "bench rc=$?"
cat gpurun_out/r2u_ln_bench.log
for i in 1 2; do for v in 3 5; do
  DDIT_LN=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2u_step_ln${v}_$i.log 2>&1
  echo "LN=$v run $i: $(tail -1 gpurun_out/r2u_step_ln${v}_$i.log | cut -c1-90)"
done; done
