# final bench (the driver's default N=1 command) + the ncu launch list of the same command without emulation
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
start=$(date +%s)
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$? elapsed=$(( $(date +%s) - start ))s
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/bench_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --emulate-pp 0 > gpurun_out/bench_ncu.log 2>&1; echo ncu rc=$?
