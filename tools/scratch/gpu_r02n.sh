mkdir -p gpurun_out
for m in 500 1000; do
for v in "H2D_SMALL_ITEMS=1" "H2D_SMALL_A=0" "H2D_SMALL_ITEMS=0"; do
  for d in "--balanced" "--balanced --directed" "--balanced --nmax 500"; do
  echo "$v $d m=$m" >> gpurun_out/adsym_n.jsonl
  env $v timeout 600 python tools/scratch/adsym_probe.py --m $m $d >> gpurun_out/adsym_n.jsonl 2>> gpurun_out/adsym_n.err
  done
done
done
