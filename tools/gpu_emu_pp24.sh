# emulated PP=2 and PP=4 (green partitions), 1F1B / BF / BFW at J0 sigma {0, 0.5} and J2 sigma 0.5
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for n in 2 4; do
  timeout 1500 python bench.py --emulate-only --emulate-pp $n --compare-jitter J0,J2 --sigmas 0.5 --steps 3 --warmup 3 > gpurun_out/emu_pp$n.json 2> gpurun_out/emu_pp$n.err; echo pp$n rc=$?; tail -1 gpurun_out/emu_pp$n.err
done
