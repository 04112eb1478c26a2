# round-end rehearsal: what the driver runs (smoke, pytest -m gpu, default bench) + the ncu launch list
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_all.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/gpu_all.log
start=$(date +%s)
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$? elapsed=$(( $(date +%s) - start ))s
timeout 900 python bench.py --impl reference > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 16000 --csv --log-file gpurun_out/bench_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --emulate-pp 0 > gpurun_out/bench_ncu.log 2>&1; echo ncu rc=$?
