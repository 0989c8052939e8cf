mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_s1" -s 4 -c 2 -o gpurun_out/r21_fuse python tools/frame_once.py B 3 > gpurun_out/r21_ncu.log 2>&1
