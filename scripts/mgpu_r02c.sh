# 4-GPU box, round-2 second-session build: rank invariance at N = 1, 2, 4, 8
# (8 = two ranks per GPU over CUDA-IPC peers) and the 8-rank bench line.
export OMP_NUM_THREADS=4
rm -f gpurun_out/mgpu_c.log
for n in 1 2 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) scripts/rank_invariance.py --out gpurun_out/rankinv_c_$n.npz > gpurun_out/rankinv_c_$n.log 2>&1
  echo "rankinv n=$n exit=$?" >> gpurun_out/mgpu_c.log
done
python scripts/rank_invariance.py --compare 'gpurun_out/rankinv_c_*.npz' > gpurun_out/rankinv_c_compare.json 2>&1; echo "compare exit=$?" >> gpurun_out/mgpu_c.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29608 bench.py --gpus 8 --steps 3 --warmup 3 --no-configs > gpurun_out/bench_c_n8.json 2> gpurun_out/bench_c_n8.err
echo "bench n=8 exit=$?" >> gpurun_out/mgpu_c.log
