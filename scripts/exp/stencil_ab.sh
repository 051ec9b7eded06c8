timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "stencil or laplace or arnoldi_config3 or rank_count" > gpurun_out/st_test.log 2>&1; echo "test exit=$?" >> gpurun_out/st.log
for v in tma smem; do KLS_STENCIL=$v python scripts/kprobe.py --j 10 --reps 20 > gpurun_out/st_$v.json 2>&1; done
ncu --set full --clock-control none -k regex:"stencil7_tma" -c 1 -f -o gpurun_out/st_tma python scripts/kprobe.py --j 10 --reps 1 > /dev/null 2>&1; echo "ncu exit=$?" >> gpurun_out/st.log
