# per-op breakdown, bench launch list, full capture of the stage GEMMs
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/op_times.py 4 > gpurun_out/op_times.txt 2>&1; echo op_times rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
  --log-file gpurun_out/bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_ncu.log 2>&1; echo ncu-list rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 30 -c 10 \
  -o gpurun_out/gemm_full python tools/prof_gemm.py > gpurun_out/gemm_full.log 2>&1; echo ncu-full rc=$?
ls -la gpurun_out
