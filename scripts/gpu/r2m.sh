set -x
timeout 300 python scripts/gemm_bench.py 2>&1 | grep "graph" > gpurun_out/r2m_gemm.log 2>&1
for b in 3 4; do DDIT_LIB=paper_2506_13497_b200/libddit_red$b.so timeout 300 python scripts/gemm_bench.py 2>&1 | grep "graph" | sed "s/^/bufs$b /" >> gpurun_out/r2m_gemm.log; done
timeout 300 python scripts/gemm_bench.py 2>&1 | grep "graph" | sed "s/^/again /" >> gpurun_out/r2m_gemm.log 2>&1
cat gpurun_out/r2m_gemm.log
