# historical (round 1 / early round 2): the x rebuild and PK_REBUILD_LOG2 were removed when the fast walks moved to exact grid-rounded states; kept to document profiles/r02_accuracy_*_rb*.txt
# speed and accuracy of the fast real walk vs the state rebuild period
O=gpurun_out
for rb in 0 6 7 8 10; do
  PK_REBUILD_LOG2=$rb timeout 300 python bench.py --no-cpu-baseline --steps 3 > $O/rb_$rb.json 2>/dev/null
  PK_REBUILD_LOG2=$rb timeout 300 python bench.py --n 36 --no-cpu-baseline --steps 3 > $O/rb36_$rb.json 2>/dev/null
done
