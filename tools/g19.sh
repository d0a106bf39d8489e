O=gpurun_out; mkdir -p $O
for v in 0 1; do for n in 32 36 40; do
  PK_DENSE_VARIANT=$v timeout 200 python bench.py --no-extra --n $n --policy qq --steps 3 --warmup 2 --no-cpu-baseline > $O/g19_qq_v${v}_$n.json 2>/dev/null
done; done
