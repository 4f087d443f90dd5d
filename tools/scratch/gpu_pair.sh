timeout 900 python -m pytest tests/test_gpu_symmetric.py tests/test_gpu_p2p_paths.py -q -x > gpurun_out/pair_tests.log 2>&1; echo rc=$? >> gpurun_out/pair_tests.log
H2D_PAIRAPPLY=1 timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e > gpurun_out/pair_bench_def.log 2>&1
for l in 1 2 3 4 5 6 7; do
H2D_PAIRAPPLY=1 H2D_PAIR_LEVELS=$l,$l timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/pair_bench_l$l.log 2>&1
done
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/dir_bench.log 2>&1
