python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -5
export RRFP_SAME_DEVICE=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --model mm --layers 4 --mb 8 --steps 2 --warmup 3 --no-compare --no-cpu-baseline > gpurun_out/bd_mm.json 2> gpurun_out/bd_mm.err; echo mm rc=$?
tail -c 700 gpurun_out/bd_mm.json; grep -i "error\|Traceback" gpurun_out/bd_mm.err | tail -5
