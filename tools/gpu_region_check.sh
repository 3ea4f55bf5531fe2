python -m pytest tests/test_gpu_regions.py tests/test_gpu_parity.py tests/test_gpu_cta.py -x -q 2>&1 | tail -3
JV_CRIT_DUMP=gpurun_out/crit_c2_factor_$1.npz python tools/region_crit.py c2 factor 2>&1 | tail -1
JV_CRIT_DUMP=gpurun_out/crit_c2_fwd_$1.npz python tools/region_crit.py c2 fwd 2>&1 | tail -1
python bench.py --config ${2:-c2} > gpurun_out/bench_${2:-c2}_$1.json 2> gpurun_out/bench_${2:-c2}_$1.err
python tools/bench_brief.py gpurun_out/bench_${2:-c2}_$1.json
