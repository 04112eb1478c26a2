# emulated PP=8 variants: W split "all", and the J3 jitter preset on top of sigma
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python bench.py --emulate-only --emulate-pp 8 --steps 3 --warmup 3 --sigmas 0.5 --w-split all \
  > gpurun_out/emu_all.json 2> gpurun_out/emu_all.err; echo rc=$?
timeout 900 python bench.py --emulate-only --emulate-pp 8 --steps 3 --warmup 3 --sigmas 0.5 --compare-jitter J3 \
  > gpurun_out/emu_j3.json 2> gpurun_out/emu_j3.err; echo rc=$?
