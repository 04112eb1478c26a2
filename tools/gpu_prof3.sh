python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
  --log-file gpurun_out/bench_launches2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --emulate-pp 0 \
  > gpurun_out/bench_ncu2.log 2>&1; echo ncu-list rc=$?
