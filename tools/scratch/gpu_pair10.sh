for l in "1,7" "1,1" "2,2" "3,3" "4,4" "5,5" "6,6" "7,7"; do
H2D_PAIRAPPLY=1 H2D_PAIR_LEVELS=$l timeout 120 python tools/scratch/pair_levels_probe.py c1 >> gpurun_out/p10.log 2>&1
H2D_PAIRAPPLY=1 H2D_PAIR_LEVELS=$l timeout 120 python tools/scratch/pair_levels_probe.py c2 >> gpurun_out/p10.log 2>&1
done
