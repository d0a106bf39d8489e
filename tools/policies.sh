# dense real n=36 under every accumulator policy (paper Table 3 analogue)
O=gpurun_out
for p in dd kahan dq qq; do
  timeout 300 python bench.py --n 36 --policy $p --no-cpu-baseline --steps 3 > $O/pol_$p.json 2> $O/pol_$p.err
done
