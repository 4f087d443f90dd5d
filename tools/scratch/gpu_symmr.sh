timeout 900 python -m pytest tests/test_gpu_symmetric.py tests/test_gpu_comm.py -q -x > gpurun_out/symmr_tests.log 2>&1; echo rc=$? >> gpurun_out/symmr_tests.log
timeout 900 python bench.py --config c5 --symmetric --rank-slice 0 --slice-world 8 --steps 10 --warmup 2 > gpurun_out/symmr_c5slice.log 2>&1
timeout 900 python bench.py --config c5 --rank-slice 0 --slice-world 8 --steps 10 --warmup 2 > gpurun_out/dir_c5slice.log 2>&1
