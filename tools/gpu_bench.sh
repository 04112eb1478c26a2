python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
start=$(date +%s)
timeout 1500 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$? elapsed=$(( $(date +%s) - start ))s
tail -3 gpurun_out/bench.err
