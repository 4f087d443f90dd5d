B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants"
for v in base p2pminb4 p2pminb5; do
  L=""; [ $v != base ] && L="H2D_LIBRARY=tools/scratch/lib_$v.so"
  env $L timeout 300 $B > gpurun_out/p2p5_$v.log 2>&1
  env $L timeout 300 python bench.py --symmetric --steps 10 --warmup 3 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/p2p5_sym_$v.log 2>&1
done
