# ncu --set full of one layer's twelve stage GEMMs -> profiles/gemm_traffic.json (bench roofline.traffic)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 36 -c 12 -o gpurun_out/gemm_full -f python tools/prof_gemm.py > gpurun_out/gemm_full.log 2>&1; echo ncu rc=$?
