# final evidence batch with the register-modulation LN: step launch list, DoP sweep (144p-360p x51), two benches
set -x
K='regex:gemm|fmha|ln_mod|temporal|final_layer|patch_embed|gemv|modulation|timestep'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 700 -c 569 --csv --log-file gpurun_out/launches_r02i.csv python scripts/profile_step.py 240p 3 > /dev/null 2>&1; echo "launches rc=$?"
python scripts/launch_summary.py gpurun_out/launches_r02i.csv | head -12
timeout 1800 python scripts/dop_sweep.py --out gpurun_out/r02i_dop_sweep.json > gpurun_out/r02i_dop_sweep.log 2>&1; echo "sweep rc=$?"
tail -15 gpurun_out/r02i_dop_sweep.log
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02i_bench_$i.log 2>&1; tail -1 gpurun_out/r02i_bench_$i.log | cut -c1-120; done
