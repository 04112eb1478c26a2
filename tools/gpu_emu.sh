python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --emulate-pp ${EMU:-8} --sigmas ${SIGMAS:-0.5} --compare-jitter ${CJ:-J0} > gpurun_out/bench_emu.json 2> gpurun_out/bench_emu.err; echo rc=$?
grep -i "emulated\|error" gpurun_out/bench_emu.err | tail -12
