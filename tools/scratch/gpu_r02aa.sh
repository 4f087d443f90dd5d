mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_p2p_paths.py tests/test_gpu_parity.py -x -q > gpurun_out/aa_tests.log 2>&1; echo rc=$? >> gpurun_out/aa_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-c4 --multi-rhs 0 --no-cpu-baseline --no-e2e > gpurun_out/aa_bench.log 2>&1
H2D_P2P_R3ROWS=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-c4 --multi-rhs 0 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/aa_bench_r3rows.log 2>&1
H2D_P2P_SERIAL=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"p2p_warp" -c 3 -o gpurun_out/r02aa_p2p python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c4 --no-variants --multi-rhs 0 --no-e2e > gpurun_out/aa_ncu.log 2>&1; echo rc=$? >> gpurun_out/aa_ncu.log
