mkdir -p gpurun_out
for lib in "" "_ab/dual3.so" "_ab/dual3b.so"; do
  H2D_LIBRARY=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-c4 --multi-rhs 0 --no-cpu-baseline --no-e2e --symmetric > gpurun_out/u_sym_$(basename "x$lib").log 2>&1
  H2D_LIBRARY=$lib timeout 600 python tools/scratch/adsym_probe.py >> gpurun_out/u_adsym_$(basename "x$lib").jsonl 2>&1
done
