timeout 900 python -m pytest tests/test_gpu_p2p_paths.py tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_rbf_gmres.py tests/test_gpu_adaptive.py -q -x > gpurun_out/p2p2_tests.log 2>&1; echo rc=$? >> gpurun_out/p2p2_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-variants --no-e2e > gpurun_out/p2p2_bench.log 2>&1
