# C5 8-way: pass 1 builds every rank slice with the geometric partition and saves its leaf
# costs (hodlr2d_leaf_costs); pass 2 rebuilds every slice partitioned by the summed costs
# and times it.  Projected E_8 of both passes: sum the per-slice "ms_per_matvec_compute" of geo_all.jsonl / mw_all.jsonl (T1_virt) over 8 x the slowest slice.
mkdir -p gpurun_out/c5w
for g in 0 1 2 3 4 5 6 7; do
  timeout 600 python bench.py --config c5 --rank-slice $g --slice-world 8 --steps 10 --warmup 2 \
    --dump-leaf-costs gpurun_out/c5w/costs_$g.npy > gpurun_out/c5w/geo_$g.json 2> gpurun_out/c5w/geo_$g.err
done
python3 -c "import numpy as np; np.save('gpurun_out/c5w/weights.npy', sum(np.load(f'gpurun_out/c5w/costs_{g}.npy') for g in range(8)))"
for g in 0 1 2 3 4 5 6 7; do
  timeout 600 python bench.py --config c5 --rank-slice $g --slice-world 8 --steps 10 --warmup 2 \
    --leaf-weights gpurun_out/c5w/weights.npy > gpurun_out/c5w/mw_$g.json 2> gpurun_out/c5w/mw_$g.err
done
cat gpurun_out/c5w/geo_*.json > gpurun_out/c5w/geo_all.jsonl
cat gpurun_out/c5w/mw_*.json > gpurun_out/c5w/mw_all.jsonl
