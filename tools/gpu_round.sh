# one measurement round on the GPU box: GPU tests, bench (N = 1), reference arm, a gloo
# functional run of the multi-GPU code path (2 ranks sharing the GPU, C5 sub-result on C2)
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gpu_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_all.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/ref.log 2>&1; echo rc=$? >> gpurun_out/ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --dist-backend gloo --c5-min-world 2 --c5-config c2 > gpurun_out/bench_gloo2.log 2>&1; echo rc=$? >> gpurun_out/bench_gloo2.log
