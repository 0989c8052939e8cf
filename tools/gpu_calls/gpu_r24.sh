mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_s1i_v2" -s 1 -c 1 -o gpurun_out/r24_D_full python tools/frame_once.py D 1 > gpurun_out/r24_ncu_D.log 2>&1
