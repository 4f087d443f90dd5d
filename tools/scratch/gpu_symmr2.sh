timeout 900 python -m pytest tests/test_gpu_symmetric.py tests/test_gpu_comm.py -q -x > gpurun_out/symmr_tests.log 2>&1; echo rc=$? >> gpurun_out/symmr_tests.log
C5_TAG=c5sym bash tools/c5_slices.sh --symmetric
