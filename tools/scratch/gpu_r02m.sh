mkdir -p gpurun_out
for m in 1000 500; do
for v in "H2D_SMALL_ITEMS=1" "H2D_SMALL_ITEMS=0" "H2D_SMALL_A_AFTER=1"; do
  for d in "" "--directed"; do
  echo "$v $d m=$m" >> gpurun_out/adsym_m.jsonl
  env $v timeout 600 python tools/scratch/adsym_probe.py --m $m $d >> gpurun_out/adsym_m.jsonl 2>> gpurun_out/adsym_m.err
  done
done
done
