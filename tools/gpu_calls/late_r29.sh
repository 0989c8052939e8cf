mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_stage" -s 4 -c 2 -o gpurun_out/late29_C python tools/frame_once.py C 3 > gpurun_out/late29_ncu.log 2>&1
