for m in cross spatial 720; do DDIT_LIB=paper_2506_13497_b200/libddit_fmtrace.so python scripts/fmha_trace.py $m > gpurun_out/fmtrace_$m.log 2>&1; done
bash scripts/gpu/sanitize.sh
