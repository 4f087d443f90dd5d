python -m pytest tests/test_gpu_adaptive.py -q -x --durations=5 > gpurun_out/adaptive_tests.log 2>&1; echo rc=$? >> gpurun_out/adaptive_tests.log
python -m pytest tests/test_gpu_p2p_paths.py tests/test_gpu_parity.py -q -x -k "subnormal or r7" > gpurun_out/num_tests.log 2>&1; echo rc=$? >> gpurun_out/num_tests.log
for m in 500 1000; do for nm in 64 128; do
timeout 600 python bench.py --mode gmres --grid-m $m --adaptive --nmax $nm >> gpurun_out/adaptive_bench.jsonl 2>> gpurun_out/adaptive_bench.err; done; done
timeout 900 python bench.py --mode gmres --grid-m 2000 --adaptive --nmax 64 >> gpurun_out/adaptive_bench.jsonl 2>> gpurun_out/adaptive_bench.err
