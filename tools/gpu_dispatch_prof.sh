# dispatcher profile (device stamps in lane_step_kernel), runtime tests, whole-graph ncu of the lane graph, launch list
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_runtime.py -q -x > gpurun_out/runtime_tests.log 2>&1; echo runtime tests rc=$?; tail -1 gpurun_out/runtime_tests.log
timeout 600 python tools/dispatch_bench.py > gpurun_out/dispatch_bench.txt 2>&1; echo dispatch rc=$?; head -4 gpurun_out/dispatch_bench.txt
timeout 300 ncu --graph-profiling graph --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/dispatch_graph_ncu.csv python tools/ncu_dispatch.py > gpurun_out/dispatch_graph_ncu.log 2>&1; echo ncu graph rc=$?; tail -3 gpurun_out/dispatch_graph_ncu.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 16000 --csv --log-file gpurun_out/bench_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --emulate-pp 0 > gpurun_out/bench_ncu.log 2>&1; echo ncu rc=$?
