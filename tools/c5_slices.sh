# All 8 rank slices of C5 on one GPU (bench.py --rank-slice): virtual T1 and projected E_8.
# Extra arguments go to every bench.py call (e.g. --symmetric); output tag via C5_TAG.
tag=${C5_TAG:-c5s}
for g in 0 1 2 3 4 5 6 7; do
  timeout 600 python bench.py --config c5 --rank-slice $g --slice-world 8 --steps 10 --warmup 2 "$@" > gpurun_out/${tag}_$g.json 2> gpurun_out/${tag}_$g.err
done
cat gpurun_out/${tag}_*.json > gpurun_out/${tag}_all.jsonl
