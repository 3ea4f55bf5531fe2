# Round-end evidence: GPU tests, smoke, bench lines of every config with the reference arm,
# the ncu launch list of the bench command and ncu --set full of one step per config.
# Outputs under gpurun_out/ (copied to profiles/ by hand).   bash tools/final_profiles.sh [tag]
TAG=${1:-final}
python -c "import __graft_entry__ as g; g.build()" || exit 1
S=$SECONDS
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_gpu_tests_$TAG.txt 2>&1
echo "gpu tests rc=$? wall=$((SECONDS-S))"; tail -3 gpurun_out/r02_gpu_tests_$TAG.txt
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py --impl reference > gpurun_out/r02_bench_reference_c2_$TAG.json 2>/dev/null
for c in c2 c1 c3 c4 c5; do
  python bench.py --config $c > gpurun_out/r02_bench_${c}_$TAG.json 2> gpurun_out/bench_$c.err || tail -5 gpurun_out/bench_$c.err
  python tools/bench_brief.py gpurun_out/r02_bench_${c}_$TAG.json
done
# launch list of the same command (cold-cache, serialised: shares only)
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches_c2_$TAG.csv python bench.py --steps 4 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
python tools/ncu_summary.py launches gpurun_out/r02_launches_c2_$TAG.csv > gpurun_out/r02_launches_c2_$TAG.txt
head -14 gpurun_out/r02_launches_c2_$TAG.txt
# one step per config under ncu --set full
for c in c2 c3 c4 c5; do
  timeout 1200 ncu --profile-from-start off --set full --clock-control none -f \
    -o gpurun_out/r02_ncu_${c}_$TAG python tools/step_once.py $c > gpurun_out/ncu_$c.log 2>&1
  tail -1 gpurun_out/ncu_$c.log
  python tools/ncu_summary.py full gpurun_out/r02_ncu_${c}_$TAG.ncu-rep > gpurun_out/r02_ncu_full_${c}_$TAG.txt
  rm -f gpurun_out/r02_ncu_${c}_$TAG.ncu-rep
done
