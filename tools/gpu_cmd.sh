python -c "import __graft_entry__ as g; g.build()" || exit 1
S=$SECONDS; timeout 900 python bench.py > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err; echo "c2 rc=$? wall=$((SECONDS-S))"; tail -3 gpurun_out/b_c2.err
S=$SECONDS; timeout 1200 python bench.py --config c5 --steps 5 > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err; echo "c5 rc=$? wall=$((SECONDS-S))"; tail -3 gpurun_out/b_c5.err
