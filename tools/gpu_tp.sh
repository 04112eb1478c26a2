python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for i in 1 2 3 4; do timeout 600 python tools/repro_rebuild.py > gpurun_out/rr.log 2>&1; echo big rc=$?; grep -o "illegal memory access\|repro done" gpurun_out/rr.log | head -1; done
for i in 1 2; do timeout 600 python tools/config3_check.py > gpurun_out/c3.log 2>&1; echo c3 rc=$?; done
