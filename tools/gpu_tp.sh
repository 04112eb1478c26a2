python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_replay_parity.py -x -q -m gpu 2>&1 | tail -3
