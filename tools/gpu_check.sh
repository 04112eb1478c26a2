# full GPU suite + emulated PP=8 (default bench emulation settings) + dispatcher microbenchmark
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/gpu_all.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gpu_all.log
timeout 900 python bench.py --emulate-only --emulate-pp 8 --steps 3 --warmup 3 --sigmas 0.5 \
  --trace-dir gpurun_out/emu_tr > gpurun_out/emu.json 2> gpurun_out/emu.err; echo emu rc=$?
timeout 300 python tools/dispatch_bench.py > gpurun_out/dispatch.txt 2>&1; echo disp rc=$?
