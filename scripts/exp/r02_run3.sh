timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "gputest exit=$?" > gpurun_out/r.log
python scripts/rotate_probe.py > gpurun_out/rotate.log 2>&1; KLS_ROTATE=fma python scripts/rotate_probe.py >> gpurun_out/rotate.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit=$?" >> gpurun_out/r.log
