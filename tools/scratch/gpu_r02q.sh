mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_adaptive.py tests/test_gpu_p2p_paths.py tests/test_gpu_symmetric.py -x -q > gpurun_out/q_tests.log 2>&1; echo rc=$? >> gpurun_out/q_tests.log
for v in "X=1" "H2D_SMALL_A_AFTER=1" "H2D_SMALL_B1=0" "H2D_SMALL_A_AFTER=1 H2D_SMALL_B1=0"; do
  for d in "" "--directed" "--balanced --nmax 500" "--balanced --nmax 500 --directed"; do
  echo "$v $d" >> gpurun_out/q_adsym.jsonl
  env $v timeout 600 python tools/scratch/adsym_probe.py --m 1000 $d >> gpurun_out/q_adsym.jsonl 2>> gpurun_out/q_adsym.err
  done
done
