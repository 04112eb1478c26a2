python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
export RRFP_SAME_DEVICE=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 2 --warmup 3 --layers 8 --mb 8 --sigmas 0.3,0.5 --compare-jitter J2 --no-cpu-baseline > gpurun_out/bd_pp4.json 2> gpurun_out/bd_pp4.err; echo pp4 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bd_pp4.json').read().strip().splitlines()[-1])
print(d['value'], d['bubble_fraction']); [print(k, v) for k, v in d['variants'].items()]"
grep -i "error\|Traceback" gpurun_out/bd_pp4.err | tail -5
