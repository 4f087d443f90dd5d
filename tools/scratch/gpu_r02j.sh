# r02j: bench (N = 1), reference arm, gloo 2-rank functional run, launch list, adaptive symmetric probe + ncu
mkdir -p gpurun_out
sed -n 7,9p tools/gpu_round.sh > /tmp/rb.sh; bash /tmp/rb.sh
sed -n 10p tools/gpu_round.sh > /tmp/rc.sh; bash /tmp/rc.sh
for m in 1000; do
  timeout 600 python tools/scratch/adsym_probe.py --m $m >> gpurun_out/adsym.jsonl 2>> gpurun_out/adsym.err
  timeout 600 python tools/scratch/adsym_probe.py --m $m --directed >> gpurun_out/adsym.jsonl 2>> gpurun_out/adsym.err
done
H2D_VERBOSE=1 timeout 600 python tools/scratch/adsym_probe.py --m 1000 --reps 2 > gpurun_out/adsym_verbose.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stage" -c 8 -o gpurun_out/r02j_adsym python tools/scratch/adsym_probe.py --m 1000 --reps 1 > gpurun_out/ncu_adsym.log 2>&1; echo rc=$? >> gpurun_out/ncu_adsym.log
