set -x
K='regex:gemm|fmha|ln_mod|temporal'
timeout 1200 ncu --set full --clock-control none --import-source on -k "$K" -s 600 -c 12 -o gpurun_out/r2l_block python scripts/profile_step.py 240p 2 > gpurun_out/r2l_ncu.log 2>&1
tail -3 gpurun_out/r2l_ncu.log
ls -la gpurun_out/
