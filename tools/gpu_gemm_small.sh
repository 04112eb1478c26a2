python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_ops.py -q -x > gpurun_out/gemm_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gemm_tests.log
timeout 900 python tools/gemm_small.py > gpurun_out/gemm_small.txt 2>&1; echo ab rc=$?; cat gpurun_out/gemm_small.txt
