# dense real K1 throughput vs order n (2^min(n-1,37)-iterate walks, KAHAN)
O=gpurun_out
for n in 16 20 24 28 32 36 40 44 48 52 56 60 63; do
  r=$(( n - 1 < 37 ? n - 1 : 37 ))
  if [ $r -ge $(( n - 1 )) ]; then RL=""; else RL="--range-log2 $r"; fi
  timeout 300 python bench.py --n $n $RL --steps 2 --warmup 3 --no-cpu-baseline > $O/sweep_n$n.json 2>/dev/null
done
