# one measurement round on the GPU box: GPU tests, bench (N = 1), reference arm, a gloo
# functional run of the multi-GPU code path (2 ranks sharing the GPU, C5 sub-result on C2),
# the ncu launch list of the default bench (build and matvec launches: -c 3000) and ncu --set
# full captures of the C3 / C4 kernels
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gpu_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/ref.log 2>&1; echo rc=$? >> gpurun_out/ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --dist-backend gloo --c5-min-world 2 --c5-config c2 > gpurun_out/bench_gloo2.log 2>&1; echo rc=$? >> gpurun_out/bench_gloo2.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo rc=$? >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stageA_tma|stageB_tma|p2p_warp" -c 4 -o gpurun_out/r02am_c3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c4 --no-variants --multi-rhs 0 --no-e2e > gpurun_out/ncu_c3.log 2>&1; echo rc=$? >> gpurun_out/ncu_c3.log
timeout 900 ncu --set full --clock-control none -k regex:"stageA_tma|stageB_tma" -c 2 -o gpurun_out/r02am_c4 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-variants --multi-rhs 0 --no-e2e > gpurun_out/ncu_c4.log 2>&1; echo rc=$? >> gpurun_out/ncu_c4.log
