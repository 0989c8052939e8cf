mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_s1_v2|k_s1_exact" -s 2 -c 2 -o gpurun_out/late56_Bq python tools/frame_once.py Bq 2 > gpurun_out/late56_ncu.log 2>&1
