python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
python tools/colsum_ab.py
for i in 1 2; do
  RRFP_COLSUM_EPI=0 timeout 600 python bench.py --emulate-pp 0 --no-cpu-baseline --steps 8 > gpurun_out/cs_off_$i.json 2>/dev/null
  timeout 600 python bench.py --emulate-pp 0 --no-cpu-baseline --steps 8 > gpurun_out/cs_on_$i.json 2>/dev/null
done
for f in gpurun_out/cs_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['clocks']['sm_mhz'], d['task_us'])"; done
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k emulated > gpurun_out/emu_test.log 2>&1; echo emu test rc=$?; tail -1 gpurun_out/emu_test.log
