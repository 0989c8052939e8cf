mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_s1i_v2" -s 1 -c 1 -o gpurun_out/late47_D python tools/frame_once.py D 2 > gpurun_out/late47_ncu.log 2>&1
