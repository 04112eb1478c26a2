# half-layer split: parity tests, then emulated PP=8
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_model.py -q -x -k "half or green" > gpurun_out/t.log 2>&1; echo rc=$?; tail -3 gpurun_out/t.log
timeout 900 python bench.py --emulate-only --emulate-pp 8 --steps 3 --warmup 3 --sigmas 0.5 --split half \
  --trace-dir gpurun_out/emu_tr_half > gpurun_out/emu_half.json 2> gpurun_out/emu_half.err; echo rc=$?
