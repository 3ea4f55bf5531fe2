# spmv kernel comparison on c2: stream kernel vs the persistent bulk kernel's ring shapes
# (JV_SPMV_CFG), back to back and right after a backward sweep (cold L2, as in the bench step)
python -m pytest tests/test_gpu_spmv.py -q -x 2>&1 | tail -3
JV_SPMV_IMPL=0 python tools/spmv_step.py 2>&1 | tail -1 | sed "s/^/stream  /"
for c in 0 1 2 3 4 5 6 7; do
  JV_SPMV_IMPL=1 JV_SPMV_CFG=$c python tools/spmv_step.py 2>&1 | tail -1 | sed "s/^/bulk cfg$c  /"
done
