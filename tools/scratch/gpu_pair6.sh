timeout 600 python -m pytest tests/test_gpu_symmetric.py -q -x > gpurun_out/p6_tests.log 2>&1; echo rc=$? >> gpurun_out/p6_tests.log
H2D_PAIRAPPLY=1 timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/p6_all.log 2>&1
H2D_PAIRAPPLY=1 H2D_P2P_SERIAL=1 timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/p6_all_serial.log 2>&1
for l in 1 3 5 6 7; do
H2D_PAIRAPPLY=1 H2D_PAIR_LEVELS=$l,$l timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/p6_l$l.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_comm.py tests/test_gpu_adaptive.py -q -x > gpurun_out/p6_tests2.log 2>&1; echo rc=$? >> gpurun_out/p6_tests2.log
C5_TAG=c5sym3 bash tools/c5_slices.sh --symmetric
