# round-2 final measurement batch: bench (driver defaults), step launch list, ncu full of one block,
# config-5 trace replay (profile best of 5) and config 4
set -x
timeout 900 python bench.py > gpurun_out/r2t_bench.log 2>&1
K='regex:gemm|fmha|ln_mod|temporal|final_layer|patch_embed|gemv|modulation|timestep'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 700 -c 569 --csv --log-file gpurun_out/r2t_launches.csv python scripts/profile_step.py 240p 3 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/r2t_launches.csv > gpurun_out/r2t_launch_summary.txt
K2='regex:gemm|fmha|ln_mod|temporal'
timeout 1200 ncu --set full --clock-control none --import-source on -k "$K2" -s 600 -c 12 -o gpurun_out/r2t_block python scripts/profile_step.py 240p 2 > gpurun_out/r2t_ncu.log 2>&1
timeout 1800 python scripts/trace_replay.py --out gpurun_out/r2t_trace_replay_c5.json > gpurun_out/r2t_trace_replay.log 2>&1
timeout 900 python scripts/config4.py --out gpurun_out/r2t_config4.json > gpurun_out/r2t_config4.log 2>&1
cat gpurun_out/r2t_launch_summary.txt | head -16; tail -c 600 gpurun_out/r2t_bench.log; grep -E "B values|predicted|replayed" gpurun_out/r2t_trace_replay.log | cut -c1-160
