O=gpurun_out; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dense_f64_chunks -s 3 -c 1 -o $O/g39_k1 python bench.py --no-extra --steps 1 --warmup 3 --range-log2 36 --no-cpu-baseline > $O/g39_ncu_k1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/g39_launches_dense40.csv python bench.py --no-extra --steps 2 --warmup 3 --no-cpu-baseline > $O/g39_ncu_launch.log 2>&1
