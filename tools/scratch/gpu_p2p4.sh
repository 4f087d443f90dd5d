B="python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants"
H2D_P2P_SERIAL=1 timeout 300 $B > gpurun_out/p2p4_serial.log 2>&1
H2D_P2P_SERIAL=1 timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:p2p --csv --log-file gpurun_out/p2p4_serial_ncu.csv $B > gpurun_out/p2p4_ncu.log 2>&1
H2D_P2P_SERIAL=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:p2p_warp_kernel --launch-skip 2 -c 1 -o gpurun_out/p2p4_full $B > gpurun_out/p2p4_full.log 2>&1
