timeout 900 python -m pytest tests/test_gpu_p2p_paths.py tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_rbf_gmres.py tests/test_gpu_adaptive.py tests/test_gpu_fullsize_parity.py -q -x -k "not c4_oracle and not c5_rank_slice_oracle" > gpurun_out/p2p3_tests.log 2>&1; echo rc=$? >> gpurun_out/p2p3_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e > gpurun_out/p2p3_bench.log 2>&1
timeout 300 python bench.py --symmetric --steps 20 --warmup 5 --no-cpu-baseline --no-c4 --multi-rhs 0 --no-e2e --no-variants > gpurun_out/p2p3_bench_sym.log 2>&1
timeout 600 python bench.py --mode gmres --grid-m 1000 --adaptive --nmax 64 --symmetric > gpurun_out/p2p3_adsym.jsonl 2>&1
