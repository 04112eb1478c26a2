python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
export RRFP_SAME_DEVICE=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 2 --warmup 3 --layers 4 --mb 8 --sigma 0.3 > gpurun_out/bd_pp2.json 2> gpurun_out/bd_pp2.err; echo pp2 rc=$?
tail -c 1500 gpurun_out/bd_pp2.json; grep -i error gpurun_out/bd_pp2.err | tail -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --tp 2 --model 7b --steps 2 --warmup 3 --layers 4 --mb 4 --no-compare > gpurun_out/bd_tp.json 2> gpurun_out/bd_tp.err; echo tp rc=$?
tail -c 1500 gpurun_out/bd_tp.json; grep -i error gpurun_out/bd_tp.err | tail -5
unset RRFP_SAME_DEVICE
timeout 600 python bench.py --impl reference --gpus 8 --steps 2 --warmup 1 > gpurun_out/bd_ref.json 2>&1; echo ref rc=$?; tail -c 800 gpurun_out/bd_ref.json
