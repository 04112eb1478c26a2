# dispatcher: runtime tests + spin-body profile + GPT bench step-kernel profile (noinline cold paths)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_replay_parity.py -q -x > gpurun_out/runtime_tests.log 2>&1; echo runtime tests rc=$?; tail -1 gpurun_out/runtime_tests.log
timeout 600 python tools/dispatch_bench.py > gpurun_out/dispatch_bench.txt 2>&1; echo dispatch rc=$?; head -4 gpurun_out/dispatch_bench.txt | cut -c1-400
timeout 900 python bench.py --emulate-pp 0 --no-cpu-baseline --steps 5 > gpurun_out/bench_pf.json 2>/dev/null; echo bench rc=$?
python -c "import json; d=json.loads(open('gpurun_out/bench_pf.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['dispatch'])"
