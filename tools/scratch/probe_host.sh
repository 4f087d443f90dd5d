nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"; free -g; df -h /tmp /dev/shm $GRAFT_REPO_ROOT | cat; cat /sys/fs/cgroup/cpu.max 2>/dev/null; cat /sys/fs/cgroup/memory.max 2>/dev/null; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python - <<'PY'
import time, numpy as np, sys
sys.path.insert(0, '.')
import oracle, workloads as W
print('threads', oracle.max_threads())
cfg = W.CONFIGS['c3']
pts = W.config_points(cfg)
t=time.time()
o = oracle.Operator(pts, cfg.kernel, cfg.leaf_size, cfg.tol, c=cfg.c, scale=cfg.scale, shift=cfg.shift, box_lo=cfg.box_lo, box_side=cfg.box_side)
print('c3 oracle build', time.time()-t, o.build_seconds, 'factor values', o.factor_values(), flush=True)
x = W.config_x(cfg, 0)
for i in range(3):
    t=time.time(); y=o.matvec(x); print('matvec', time.time()-t, flush=True)
oracle.set_threads(1)
t=time.time(); y=o.matvec(x); print('matvec 1 thread', time.time()-t, flush=True)
PY
free -g
