for k in rbf_phi1 rbf_phi2; do timeout 300 python bench.py --mode gmres --rbf-kernel $k 2>/dev/null | tail -1; done > gpurun_out/gmres_250000.jsonl
timeout 600 python -m pytest tests/test_gpu_rbf_gmres.py -x -q --timeout 300 2>&1 | tail -2
