mkdir -p gpurun_out
for m in 1000; do
  H2D_P2P_SERIAL=1 timeout 600 python tools/scratch/adsym_probe.py --m $m >> gpurun_out/adsym_k.jsonl 2>> gpurun_out/adsym_k.err
  H2D_P2P_SERIAL=1 timeout 600 python tools/scratch/adsym_probe.py --m $m --directed >> gpurun_out/adsym_k.jsonl 2>> gpurun_out/adsym_k.err
  H2D_SMALL_ITEMS=0 timeout 600 python tools/scratch/adsym_probe.py --m $m >> gpurun_out/adsym_k.jsonl 2>> gpurun_out/adsym_k.err
done
timeout 600 python tools/scratch/adsym_probe.py --m 500 >> gpurun_out/adsym_k.jsonl 2>> gpurun_out/adsym_k.err
H2D_P2P_SERIAL=1 timeout 600 python tools/scratch/adsym_probe.py --m 500 >> gpurun_out/adsym_k.jsonl 2>> gpurun_out/adsym_k.err
timeout 900 ncu --set full --clock-control none -k regex:"p2p" -c 6 -o gpurun_out/r02k_adsym_p2p python tools/scratch/adsym_probe.py --m 1000 --reps 1 > gpurun_out/ncu_adsym_p2p.log 2>&1; echo rc=$? >> gpurun_out/ncu_adsym_p2p.log
