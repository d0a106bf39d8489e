O=gpurun_out; mkdir -p $O
for v in 0 1 2 3; do
  for n in 36 40; do
    PK_DENSE_VARIANT=$v timeout 120 python bench.py --n $n --steps 3 --warmup 2 --no-cpu-baseline > $O/g12_dense_v${v}_$n.json 2>/dev/null
  done
  PK_DENSE_VARIANT=$v timeout 120 python bench.py --n 48 --steps 2 --warmup 2 --range-log2 41 --no-cpu-baseline > $O/g12_dense_v${v}_48.json 2>/dev/null
done
for v in 2 3 4 5; do
  for n in 28 32 36; do
    PK_C128_VARIANT=$v timeout 120 python bench.py --workload haar --n $n --steps 3 --warmup 2 --no-cpu-baseline > $O/g12_haar_v${v}_$n.json 2>/dev/null
  done
done
for v in 2 3; do
  for n in 41 48; do
    PK_C128_VARIANT=$v timeout 150 python bench.py --workload haar --n $n --steps 2 --warmup 2 --range-log2 38 --no-cpu-baseline > $O/g12_pair_v${v}_$n.json 2>/dev/null
  done
done
PK_BENCH_SHARE_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --n 36 --steps 2 --warmup 3 --no-cpu-baseline > $O/g12_torchrun2_shared.json 2> $O/g12_torchrun2_shared.err
timeout 600 python -m pytest tests/test_gpu_schedules.py -m gpu -q > $O/g12_pytest_schedules.txt 2>&1
