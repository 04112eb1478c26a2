python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
