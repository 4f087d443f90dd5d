mkdir -p gpurun_out
for v in "X=1" "H2D_DUAL_NS=4"; do
  for d in "" "--balanced --nmax 500"; do
  echo "$v $d" >> gpurun_out/r_adsym.jsonl
  env $v timeout 600 python tools/scratch/adsym_probe.py --m 1000 $d >> gpurun_out/r_adsym.jsonl 2>> gpurun_out/r_adsym.err
  done
  env $v timeout 600 python bench.py --steps 20 --warmup 5 --no-c4 --multi-rhs 0 --no-cpu-baseline --no-e2e --symmetric > gpurun_out/r_sym_$(echo $v | tr '= ' '__').log 2>&1
done
