# backward launch list (device time per kernel) + full capture of the main backward kernel
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/attn_bwd_launches.csv python tools/attn_bench.py --bwd --only-ours > /dev/null 2>&1; echo list rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fmha_bwd -s 3 -c 1 -o gpurun_out/attn_bwd_prof -f python tools/attn_bench.py --bwd --only-ours > gpurun_out/attn_bwd_ncu.log 2>&1; echo ncu rc=$?
