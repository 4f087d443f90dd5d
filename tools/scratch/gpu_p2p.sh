timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-variants --no-e2e > gpurun_out/p2p_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:p2p_warp -c 2 -o gpurun_out/p2p_warp python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c4 --no-variants --multi-rhs 0 --no-e2e > gpurun_out/ncu_p2p.log 2>&1
