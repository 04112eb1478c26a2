python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_dist.py -x -q 2>&1 | tail -2
timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --emulate-pp ${EMU:-4} --sigmas 0.5 > gpurun_out/bench_emu.json 2> gpurun_out/bench_emu.err; echo rc=$?
grep -i "emulated\|error" gpurun_out/bench_emu.err | tail -12
