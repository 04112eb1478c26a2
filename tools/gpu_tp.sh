python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_model.py -q -k green > gpurun_out/t.log 2>&1; echo rc=$?; tail -3 gpurun_out/t.log
timeout 1500 python bench.py --emulate-only --emulate-pp 8 --steps 3 --warmup 3 --sigmas 0.5 > gpurun_out/emu_green.json 2> gpurun_out/emu_green.err; echo emu rc=$?
tail -4 gpurun_out/emu_green.err
