python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 30 -c 10 \
  -o gpurun_out/gemm_full2 python tools/prof_gemm.py > gpurun_out/gemm_full2.log 2>&1; echo ncu rc=$?
