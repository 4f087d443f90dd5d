mkdir -p gpurun_out
for v in "X=1" "H2D_DUAL_NOROW=1"; do
  env $v timeout 600 python bench.py --steps 20 --warmup 5 --no-c4 --multi-rhs 0 --no-cpu-baseline --no-e2e --symmetric > gpurun_out/ac_sym_$(echo $v | tr '= ' '__').log 2>&1
  env $v H2D_P2P_SERIAL=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-c4 --multi-rhs 0 --no-cpu-baseline --no-e2e --symmetric > gpurun_out/ac_symser_$(echo $v | tr '= ' '__').log 2>&1
  env $v timeout 600 python tools/scratch/adsym_probe.py >> gpurun_out/ac_adsym_$(echo $v | tr '= ' '__').jsonl 2>&1
done
