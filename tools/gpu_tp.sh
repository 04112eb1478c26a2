python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1500 python bench.py --emulate-only --emulate-pp 8 --steps 3 --warmup 3 --sigmas 0,0.1,0.2,0.3,0.4,0.5 > gpurun_out/emu_sweep.json 2> gpurun_out/emu_sweep.err; echo rc=$?
tail -3 gpurun_out/emu_sweep.err
