for l in 5 7; do
H2D_PAIRAPPLY=1 H2D_PAIR_LEVELS=$l,$l timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/pair_red_l$l.log 2>&1
H2D_LIBRARY=tools/scratch/libhodlr2d_nored.so H2D_PAIRAPPLY=1 H2D_PAIR_LEVELS=$l,$l timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/pair_nored_l$l.log 2>&1
done
H2D_PAIRAPPLY=1 H2D_PAIR_LEVELS=7,7 timeout 600 ncu --set full --clock-control none --import-source on -k regex:pair_apply -c 1 -o gpurun_out/pair2_l7 python bench.py --symmetric --steps 2 --warmup 1 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/ncu2_l7.log 2>&1
