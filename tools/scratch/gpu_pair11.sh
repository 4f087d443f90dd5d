B="python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants"
for v in base diag1 diag3; do
  L=""; [ $v != base ] && L="H2D_LIBRARY=tools/scratch/lib_$v.so"
  for lv in "7,7" "5,5" "1,7"; do
    env $L H2D_PAIRAPPLY=1 H2D_P2P_SERIAL=1 H2D_PAIR_LEVELS=$lv timeout 120 $B > gpurun_out/p11_${v}_${lv/,/_}.log 2>&1
  done
done
