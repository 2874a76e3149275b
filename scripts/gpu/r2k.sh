set -x
python -m pytest tests/test_attention_gpu.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/r2k_unit.log
timeout 300 python scripts/attn_bench.py > gpurun_out/r2k_attn.log 2>&1
for m in cross spatial 720; do DDIT_LIB=paper_2506_13497_b200/libddit_fmtrace.so timeout 300 python scripts/fmha_trace.py $m > gpurun_out/r2k_fmtrace_$m.log 2>&1; done
cat gpurun_out/r2k_unit.log gpurun_out/r2k_attn.log
