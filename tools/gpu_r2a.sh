# round-2 check of the restored tree: smoke, the GPU suite, the default bench
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r2a_smoke.log
timeout 2100 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2a_gpu.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2a_gpu.log
start=$(date +%s)
timeout 1500 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo bench rc=$? elapsed=$(( $(date +%s) - start ))s
