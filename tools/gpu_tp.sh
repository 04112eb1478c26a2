python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_dist.py -q -k second > gpurun_out/t.log 2>&1; echo rc=$?; tail -3 gpurun_out/t.log
