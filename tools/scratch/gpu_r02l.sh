mkdir -p gpurun_out
for c in 1 2 3; do
  H2D_P2P_LIST_CTAS=$c timeout 600 python tools/scratch/adsym_probe.py --m 1000 >> gpurun_out/adsym_l.jsonl 2>> gpurun_out/adsym_l.err
done
H2D_P2P_LIST_CTAS=1 timeout 600 python tools/scratch/adsym_probe.py --m 1000 --directed >> gpurun_out/adsym_l.jsonl 2>> gpurun_out/adsym_l.err
H2D_SMALL_ITEMS=0 timeout 600 python tools/scratch/adsym_probe.py --m 1000 >> gpurun_out/adsym_l.jsonl 2>> gpurun_out/adsym_l.err
timeout 600 python tools/scratch/adsym_probe.py --m 500 >> gpurun_out/adsym_l.jsonl 2>> gpurun_out/adsym_l.err
timeout 600 python tools/scratch/adsym_probe.py --m 2000 >> gpurun_out/adsym_l.jsonl 2>> gpurun_out/adsym_l.err
