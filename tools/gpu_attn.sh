# attention core: parity tests + timing vs cuDNN (+ optional ncu capture)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests/test_gpu_attn.py -q -x > gpurun_out/attn_tests.log 2>&1; echo tests rc=$?; tail -15 gpurun_out/attn_tests.log
timeout 300 python tools/attn_bench.py ${ATTN_ARGS} > gpurun_out/attn_bench.json 2> gpurun_out/attn_bench.err; echo bench rc=$?; cat gpurun_out/attn_bench.json; tail -3 gpurun_out/attn_bench.err
if [ -n "$ATTN_NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fmha -s 5 -c 1 -o gpurun_out/attn_prof -f python tools/attn_bench.py --only-ours ${ATTN_ARGS} > gpurun_out/attn_ncu.log 2>&1; echo ncu rc=$?
fi
