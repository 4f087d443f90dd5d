set -x
python -m pytest tests/test_gpu_comm.py -v -x > gpurun_out/comm.log 2>&1; echo comm_rc=$? >> gpurun_out/comm.log
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize_parity.py --durations=15 > gpurun_out/gpu_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_all.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --dist-backend gloo > gpurun_out/bench_gloo2.log 2>&1; echo rc=$? >> gpurun_out/bench_gloo2.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02a.log 2>&1; echo rc=$? >> gpurun_out/bench_r02a.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/ref_r02a.log 2>&1; echo rc=$? >> gpurun_out/ref_r02a.log
