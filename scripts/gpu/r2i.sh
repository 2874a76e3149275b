set -x
for pp in 0 2 3 4; do DDIT_FMHA_POLY=$pp timeout 300 python scripts/attn_bench.py 2>&1 | grep "tc=True" | sed "s/^/poly$pp /" >> gpurun_out/r2i_poly.log; done
for m in cross spatial; do DDIT_LIB=paper_2506_13497_b200/libddit_fmtrace.so timeout 300 python scripts/fmha_trace.py $m > gpurun_out/r2i_fmtrace_$m.log 2>&1; done
cat gpurun_out/r2i_poly.log
