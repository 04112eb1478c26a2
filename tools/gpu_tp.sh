python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_model.py -x -q 2>&1 | tail -2
timeout 300 python tools/task_times.py 3 2>&1 | tail -2
timeout 300 python tools/task_times.py 3 bfw 2>&1 | tail -2
