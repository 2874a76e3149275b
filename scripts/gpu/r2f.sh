# round 2 run f: reduce-add residual epilogue, streaming LN, FMHA ragged-tile exps branch
set -x
python -m pytest tests/test_gemm_gpu.py tests/test_attention_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2f_unit.log
timeout 300 python scripts/attn_bench.py > gpurun_out/r2f_attn.log 2>&1
for m in cross spatial; do DDIT_LIB=paper_2506_13497_b200/libddit_fmtrace.so timeout 300 python scripts/fmha_trace.py $m > gpurun_out/r2f_fmtrace_$m.log 2>&1; done
DDIT_LN=1 timeout 600 python scripts/ab_step.py 240p ln1 > gpurun_out/r2f_ab_ln1.log 2>&1
DDIT_LN=3 timeout 600 python scripts/ab_step.py 240p ln3 > gpurun_out/r2f_ab_ln3.log 2>&1
timeout 1500 python -m pytest tests/test_parity_configs_gpu.py tests/test_step_gpu.py tests/test_group_gpu.py -m gpu -x -q -s 2>&1 | grep -E "relL2|diff|passed|failed|Error|error" | tail -60 > gpurun_out/r2f_parity.log
K='regex:gemm|fmha|ln_mod|temporal|final_layer|patch_embed|gemv|modulation|timestep'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 700 -c 569 --csv --log-file gpurun_out/r2f_launches.csv python scripts/profile_step.py 240p 3 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/r2f_launches.csv > gpurun_out/r2f_launch_summary.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 60 python scripts/sanitize_case.py > gpurun_out/r2f_san_racecheck.log 2>&1
tail -3 gpurun_out/r2f_san_racecheck.log
cat gpurun_out/r2f_unit.log gpurun_out/r2f_attn.log gpurun_out/r2f_ab_*.log gpurun_out/r2f_parity.log gpurun_out/r2f_launch_summary.txt | tail -80
