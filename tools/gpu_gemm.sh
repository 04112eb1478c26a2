python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -5
timeout 300 python tools/gemm_ab.py 2>&1 | tee gpurun_out/gemm_ab.txt
