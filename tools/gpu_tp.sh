python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/t.log 2>&1; echo dist rc=$?; tail -1 gpurun_out/t.log
export RRFP_SAME_DEVICE=1
start=$(date +%s)
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/bd_full2.json 2> gpurun_out/bd_full2.err; echo rc=$? elapsed=$(( $(date +%s) - start ))s
grep -i "rrfp error\|OutOfMemory" gpurun_out/bd_full2.err | head -5
