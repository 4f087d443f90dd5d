mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stageA_dual|stageA_tma" -c 2 -o gpurun_out/r02ab_sym python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c4 --no-variants --multi-rhs 0 --no-e2e --symmetric > gpurun_out/ab_ncu.log 2>&1; echo rc=$? >> gpurun_out/ab_ncu.log
