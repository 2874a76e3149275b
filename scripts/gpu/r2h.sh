# round 2 run h: FMHA flat tile stream + deferred epilogue (A/B against the previous kernel)
set -x
python -m pytest tests/test_attention_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2h_unit.log
timeout 300 python scripts/attn_bench.py > gpurun_out/r2h_attn.log 2>&1
DDIT_LIB=paper_2506_13497_b200/libddit_fmold.so timeout 300 python scripts/attn_bench.py > gpurun_out/r2h_attn_old.log 2>&1
for m in cross spatial; do DDIT_LIB=paper_2506_13497_b200/libddit_fmtrace.so timeout 300 python scripts/fmha_trace.py $m > gpurun_out/r2h_fmtrace_$m.log 2>&1; done
timeout 1500 python -m pytest tests/test_step_gpu.py tests/test_parity_configs_gpu.py -m gpu -x -q -s 2>&1 | grep -E "relL2|diff|passed|failed|Error|error" | tail -40 > gpurun_out/r2h_parity.log
cat gpurun_out/r2h_unit.log gpurun_out/r2h_attn.log gpurun_out/r2h_attn_old.log gpurun_out/r2h_parity.log
