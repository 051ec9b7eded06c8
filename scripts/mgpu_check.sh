timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "gputest exit=$?" >> gpurun_out/mgpu.log
set -x
export OMP_NUM_THREADS=4
for n in 1 2 3 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500+n)) scripts/rank_invariance.py --out gpurun_out/rankinv_$n.npz > gpurun_out/rankinv_$n.log 2>&1
  echo "n=$n exit=$?" >> gpurun_out/mgpu.log
done
python scripts/rank_invariance.py --compare 'gpurun_out/rankinv_*.npz' > gpurun_out/rankinv_compare.json 2>&1; echo "compare exit=$?" >> gpurun_out/mgpu.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29600 scripts/peer_capi_check.py > gpurun_out/peer_capi_4.log 2>&1; echo "capi4 exit=$?" >> gpurun_out/mgpu.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29601 scripts/peer_capi_check.py > gpurun_out/peer_capi_8.log 2>&1; echo "capi8 exit=$?" >> gpurun_out/mgpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29602 scripts/rank_invariance.py --out gpurun_out/rankinv_8.npz > gpurun_out/rankinv_8.log 2>&1; echo "n=8 exit=$?" >> gpurun_out/mgpu.log
python scripts/rank_invariance.py --compare 'gpurun_out/rankinv_*.npz' > gpurun_out/rankinv_compare8.json 2>&1; echo "compare8 exit=$?" >> gpurun_out/mgpu.log
