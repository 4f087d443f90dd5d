mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stage[AB]_multi" -c 2 -o gpurun_out/r02x_multi16 python bench.py --steps 14 --warmup 2 --no-cpu-baseline --no-c4 --no-variants --multi-rhs 16 --no-e2e > gpurun_out/x_ncu.log 2>&1; echo rc=$? >> gpurun_out/x_ncu.log
