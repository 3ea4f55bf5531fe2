python -c "import __graft_entry__ as g; g.build()" || exit 1
S=$SECONDS; timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.txt 2>&1; echo "rc=$? wall=$((SECONDS-S))"; tail -5 gpurun_out/gputest.txt
python -c "import __graft_entry__ as g; g.smoke()"
