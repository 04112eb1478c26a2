python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
export RRFP_SAME_DEVICE=1
start=$(date +%s)
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29554 bench.py --gpus 8 --steps 2 --warmup 3 > gpurun_out/bd_full8.json 2> gpurun_out/bd_full8.err; echo rc=$? elapsed=$(( $(date +%s) - start ))s
grep -i "rrfp error\|OutOfMemory\|Traceback" gpurun_out/bd_full8.err | head -5
