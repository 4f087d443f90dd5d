mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_async.py tests/test_gpu_api_checks.py -x -q > gpurun_out/v_tests.log 2>&1; echo rc=$? >> gpurun_out/v_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 --multi-rhs 0 --no-cpu-baseline --no-variants > gpurun_out/v_bench.log 2>&1; echo rc=$? >> gpurun_out/v_bench.log
