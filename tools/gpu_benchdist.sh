# the driver's N>1 bench command with every rank on cuda:0 (RRFP_SAME_DEVICE=1): full-size 1.3B
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
export RRFP_SAME_DEVICE=1
N=${1:-8}
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/bd_full$N.json 2> gpurun_out/bd_full$N.err; echo pp$N rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bd_full$N.json').read().strip().splitlines()[-1])
print(d['value'], d['bubble_fraction'], d['config']['layer_split'], d.get('dispatch')); [print(k, {a: b for a, b in v.items() if a != 'dispatch'}) for k, v in d['variants'].items()]"
grep -i "error\|Traceback" gpurun_out/bd_full$N.err | tail -5
