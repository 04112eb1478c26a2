# b_1 column sums in the FC2-dgrad epilogue, the N>1 bench path end to end (2 ranks on one GPU), model
# parity; then the config-5 sigma sweep at J2 on the emulated PP=8 (nominal times measured without jitter)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_ops.py -q -x > gpurun_out/gemm_tests.log 2>&1; echo gemm/ops tests rc=$?; tail -1 gpurun_out/gemm_tests.log
timeout 1500 python -m pytest tests/test_gpu_model.py tests/test_gpu_dist.py -q -x > gpurun_out/model_tests.log 2>&1; echo model/dist tests rc=$?; tail -3 gpurun_out/model_tests.log
timeout 2400 python bench.py --emulate-only --emulate-pp 8 --compare-jitter J2 --sigmas 0,0.1,0.2,0.3,0.4,0.5 --steps 3 --warmup 3 > gpurun_out/sweep_j2.json 2> gpurun_out/sweep_j2.err; echo sweep rc=$?
tail -2 gpurun_out/sweep_j2.err
