# 4-GPU box: tests, the 1-GPU bench (configs block), rank invariance at
# N = 1, 2, 3, 4 and 8 (two ranks per GPU), and the strong-scaling bench lines.
export OMP_NUM_THREADS=4
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "gputest exit=$?" >> gpurun_out/mgpu.log
timeout 1200 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench1 exit=$?" >> gpurun_out/mgpu.log
for n in 1 2 3 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) scripts/rank_invariance.py --out gpurun_out/rankinv_$n.npz > gpurun_out/rankinv_$n.log 2>&1
  echo "rankinv n=$n exit=$?" >> gpurun_out/mgpu.log
done
python scripts/rank_invariance.py --compare 'gpurun_out/rankinv_*.npz' > gpurun_out/rankinv_compare.json 2>&1; echo "compare exit=$?" >> gpurun_out/mgpu.log
for n in 2 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600+n)) bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  echo "bench n=$n exit=$?" >> gpurun_out/mgpu.log
done
