for c in 2 3; do for l in 5 7; do
H2D_PAIR_CTAS=$c H2D_PAIRAPPLY=1 H2D_PAIR_LEVELS=$l,$l timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/p3_c${c}_l$l.log 2>&1
done
H2D_PAIR_CTAS=$c H2D_PAIRAPPLY=1 timeout 120 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/p3_c${c}_all.log 2>&1
done
