timeout 900 python -m pytest tests/test_gpu_symmetric.py -q -x > gpurun_out/p12_tests.log 2>&1; echo rc=$? >> gpurun_out/p12_tests.log
H2D_PAIRAPPLY=1 timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/p12_pair.log 2>&1
timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/p12_sym.log 2>&1
