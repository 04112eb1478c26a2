python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python tools/config3_check.py 2>&1 | grep -v "^\s*File\|^\s*\^" | tail -8
