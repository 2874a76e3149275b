# round 2 run g: fixes (RED plan + late exchange attach), FMHA producer order
set -x
python -m pytest tests/test_gemm_gpu.py tests/test_attention_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2g_unit.log
timeout 300 python scripts/attn_bench.py > gpurun_out/r2g_attn.log 2>&1
for m in cross spatial; do DDIT_LIB=paper_2506_13497_b200/libddit_fmtrace.so timeout 300 python scripts/fmha_trace.py $m > gpurun_out/r2g_fmtrace_$m.log 2>&1; done
timeout 1500 python -m pytest tests/test_parity_configs_gpu.py tests/test_step_gpu.py tests/test_group_gpu.py -m gpu -x -q -s 2>&1 | grep -E "relL2|diff|passed|failed|Error|error" | tail -60 > gpurun_out/r2g_parity.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_bench.log 2>&1
cat gpurun_out/r2g_unit.log gpurun_out/r2g_attn.log gpurun_out/r2g_parity.log | tail -60; tail -c 1500 gpurun_out/r2g_bench.log
