# default bench (cuBLAS reference on the 12 GEMM shapes), then the config-5 sigma sweep at J2 on the emulated PP=8
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
start=$(date +%s)
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$? elapsed=$(( $(date +%s) - start ))s
timeout 2400 python bench.py --emulate-only --emulate-pp 8 --compare-jitter J2 --sigmas 0,0.1,0.2,0.3,0.4,0.5 --steps 3 --warmup 3 > gpurun_out/sweep_j2.json 2> gpurun_out/sweep_j2.err; echo sweep rc=$?
tail -2 gpurun_out/sweep_j2.err
