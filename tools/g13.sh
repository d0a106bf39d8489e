O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_complex.py tests/test_gpu_sparse_complex.py tests/test_gpu_batch.py tests/test_gpu_configs.py tests/test_gpu_schedules.py tests/test_gpu_edges.py -m gpu -q -x > $O/g13_pytest.txt 2>&1
for n in 28 32 36 40; do
  timeout 200 python bench.py --workload haar --n $n --steps 3 --warmup 2 --no-cpu-baseline > $O/g13_haar_$n.json 2>/dev/null
done
PK_BENCH_SHARE_GPU=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > $O/g13_torchrun2_shared.json 2> $O/g13_torchrun2_shared.err
