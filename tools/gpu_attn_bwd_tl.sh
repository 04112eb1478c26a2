# attention backward event timeline (two CTAs) + dispatcher L2-prefetch check
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 300 python tools/attn_timeline.py --bwd --cta 0 112 > gpurun_out/attn_bwd_timeline.txt 2>&1; echo timeline rc=$?
timeout 600 python tools/dispatch_bench.py > gpurun_out/dispatch_bench.txt 2>&1; echo dispatch rc=$?; head -2 gpurun_out/dispatch_bench.txt
timeout 900 python bench.py --emulate-pp 0 --no-cpu-baseline --steps 5 > gpurun_out/bench_pf.json 2>/dev/null; echo bench rc=$?
python -c "import json; d=json.loads(open('gpurun_out/bench_pf.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['dispatch'])"
