mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/z_tests.log 2>&1; echo rc=$? >> gpurun_out/y_tests.log
timeout 900 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-c4 --no-variants --no-e2e --multi-rhs 16 > gpurun_out/z_bench16.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c4 --no-variants --no-e2e --multi-rhs 8 > gpurun_out/z_bench8.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"stage[AB]_multi" -c 2 -o gpurun_out/r02z_multi16 python bench.py --steps 14 --warmup 2 --no-cpu-baseline --no-c4 --no-variants --multi-rhs 16 --no-e2e > gpurun_out/z_ncu.log 2>&1; echo rc=$? >> gpurun_out/y_ncu.log
