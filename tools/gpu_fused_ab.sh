# LN side-pass fusion + LM-head CE: parity tests, PP=1 step A/B (interleaved), dispatcher ncu probe, launch list
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x > gpurun_out/ops_tests.log 2>&1; echo ops tests rc=$?; tail -1 gpurun_out/ops_tests.log
timeout 1200 python -m pytest tests/test_gpu_model.py tests/test_gpu_dist.py -q -x > gpurun_out/model_tests.log 2>&1; echo model tests rc=$?; tail -1 gpurun_out/model_tests.log
for i in 1 2; do
  RRFP_LN_FUSED=0 RRFP_CE_FUSED=0 timeout 600 python bench.py --emulate-pp 0 --no-cpu-baseline --steps 8 > gpurun_out/ab_off_$i.json 2>/dev/null; echo off rc=$?
  timeout 600 python bench.py --emulate-pp 0 --no-cpu-baseline --steps 8 > gpurun_out/ab_on_$i.json 2>/dev/null; echo on rc=$?
done
for f in gpurun_out/ab_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['clocks']['sm_mhz'], d['task_us'])"; done
timeout 300 ncu --kernel-name regex:lane_ --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/dispatch_ncu.csv python tools/ncu_dispatch.py > gpurun_out/dispatch_ncu.log 2>&1; echo ncu dispatch rc=$?; tail -3 gpurun_out/dispatch_ncu.log
