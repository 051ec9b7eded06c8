timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "gputest exit=$?" > gpurun_out/f1.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit=$?" >> gpurun_out/f1.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv -c 700 python bench.py --steps 1 --warmup 1 --no-configs --no-cpu-baseline --no-e2e --traced 1 > gpurun_out/ncu_bench.log 2>&1; echo "launches exit=$?" >> gpurun_out/f1.log
ncu --set full --import-source on --clock-control none -k regex:"gram_tma_kernel|dcgs2_update_tma_kernel|stencil7_tma_kernel" -c 3 -f -o gpurun_out/k_r02 python scripts/exp/ncu_probe.py > gpurun_out/ncu_probe.log 2>&1; echo "full exit=$?" >> gpurun_out/f1.log
