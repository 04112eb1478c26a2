python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 300 python tools/task_times.py 4 2>&1 | tee gpurun_out/task_times.txt
timeout 300 python tools/task_times.py 4 bfw 2>&1 | tee -a gpurun_out/task_times.txt
