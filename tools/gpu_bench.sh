# default bench (the driver's N=1 command) + model-gpu tests
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_model.py -q -x > gpurun_out/model_tests.log 2>&1; echo model tests rc=$?; tail -2 gpurun_out/model_tests.log
start=$(date +%s)
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$? elapsed=$(( $(date +%s) - start ))s
tail -3 gpurun_out/bench.err
