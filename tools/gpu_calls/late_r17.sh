mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_s1_pipe" -s 2 -c 1 -o gpurun_out/r17_pipe python tools/frame_once.py B 3 > gpurun_out/r17_ncu.log 2>&1
