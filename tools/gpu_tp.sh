python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
export RRFP_SAME_DEVICE=1 RRFP_WATCHDOG=60
for i in 1 2 3; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=2953$i tools/dist_check.py bfw 2 1 > gpurun_out/dc$i.log 2>&1; echo rc=$?
grep -n "watchdog" gpurun_out/dc$i.log | head -3
done
unset RRFP_SAME_DEVICE RRFP_WATCHDOG
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_runtime.py -x -q 2>&1 | tail -3
