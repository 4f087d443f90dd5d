mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_adaptive.py tests/test_gpu_rbf_gmres.py -x -q > gpurun_out/s_tests.log 2>&1; echo rc=$? >> gpurun_out/s_tests.log
for d in "" "--directed" "--m 500" "--m 2000"; do
  echo "$d" >> gpurun_out/s_adsym.jsonl
  timeout 600 python tools/scratch/adsym_probe.py $d >> gpurun_out/s_adsym.jsonl 2>> gpurun_out/s_adsym.err
done
H2D_P2P_SERIAL=1 timeout 600 python tools/scratch/adsym_probe.py >> gpurun_out/s_adsym.jsonl 2>> gpurun_out/s_adsym.err
