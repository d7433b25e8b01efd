set -x
timeout 3000 python -m pytest tests -q -m gpu --durations=8 > gpurun_out/r2_gputest_full.log 2>&1; echo "pytest rc=$?"
tail -16 gpurun_out/r2_gputest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
