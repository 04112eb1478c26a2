python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_model.py -q 2>&1 | tail -1
