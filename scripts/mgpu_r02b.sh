# 4-GPU box, final round-2 build: multi-GPU tests, rank invariance,
# strong-scaling bench lines for DCGS2 and the CGS2 comparator.
export OMP_NUM_THREADS=4
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/gpumulti.log 2>&1; echo "gpumulti exit=$?" >> gpurun_out/mgpu.log
for n in 1 2 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) scripts/rank_invariance.py --out gpurun_out/rankinv_$n.npz > gpurun_out/rankinv_$n.log 2>&1
  echo "rankinv n=$n exit=$?" >> gpurun_out/mgpu.log
done
python scripts/rank_invariance.py --compare 'gpurun_out/rankinv_*.npz' > gpurun_out/rankinv_compare.json 2>&1; echo "compare exit=$?" >> gpurun_out/mgpu.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600+n)) bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
  echo "bench n=$n exit=$?" >> gpurun_out/mgpu.log
done
for n in 1 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700+n)) bench.py --gpus $n --scheme cgs2 --no-configs --no-cpu-baseline > gpurun_out/bench_cgs2_n$n.json 2> gpurun_out/bench_cgs2_n$n.err
  echo "bench cgs2 n=$n exit=$?" >> gpurun_out/mgpu.log
done
