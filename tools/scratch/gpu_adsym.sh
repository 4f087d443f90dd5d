timeout 600 python -m pytest tests/test_gpu_adaptive.py tests/test_gpu_symmetric.py -q -x > gpurun_out/adsym_tests.log 2>&1; echo rc=$? >> gpurun_out/adsym_tests.log
for m in 500 1000; do
timeout 600 python bench.py --mode gmres --grid-m $m --adaptive --nmax 64 --symmetric >> gpurun_out/adsym_bench.jsonl 2>> gpurun_out/adsym_bench.err
done
timeout 900 python bench.py --mode gmres --grid-m 2000 --adaptive --nmax 64 --symmetric >> gpurun_out/adsym_bench.jsonl 2>> gpurun_out/adsym_bench.err
