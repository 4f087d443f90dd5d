timeout 600 python -m pytest tests/test_gpu_symmetric.py -q -x -k "pair" > gpurun_out/p8_tests.log 2>&1; echo rc=$? >> gpurun_out/p8_tests.log
H2D_PAIRAPPLY=1 timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/p8_all.log 2>&1
H2D_PAIRAPPLY=1 H2D_P2P_SERIAL=1 timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/p8_all_serial.log 2>&1
for l in 1 2 3 4 5 6 7; do
H2D_PAIRAPPLY=1 H2D_P2P_SERIAL=1 H2D_PAIR_LEVELS=$l,$l timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/p8_l$l.log 2>&1
done
H2D_PAIRAPPLY=1 H2D_PAIR_LEVELS=7,7 timeout 600 ncu --set full --clock-control none --import-source on -k regex:pair_apply -c 1 -o gpurun_out/pair8_l7 python bench.py --symmetric --steps 2 --warmup 1 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/ncu8_l7.log 2>&1
