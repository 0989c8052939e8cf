mkdir -p gpurun_out
python bench.py > gpurun_out/late95_bench.json 2> gpurun_out/late95_bench.err
python tools/resolve_once.py B > gpurun_out/late95_resolve_B.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_resolve -c 1 -o gpurun_out/late95_resolve_B python tools/resolve_once.py B > gpurun_out/late95_ncu_resolve_B.log 2>&1
python tools/resolve_once.py A4 > gpurun_out/late95_resolve_A4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_resolve|k_downsample" -c 2 -o gpurun_out/late95_resolve_A4 python tools/resolve_once.py A4 > gpurun_out/late95_ncu_resolve_A4.log 2>&1
