mkdir -p gpurun_out
CURAST_S1=v2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_s1_v2|k_s1_exact" -c 2 -o gpurun_out/r3_v2_full python tools/frame_once.py B 1 > gpurun_out/r3_ncu.log 2>&1
ncu -i gpurun_out/r3_v2_full.ncu-rep --page source --csv --print-source sass -k regex:k_s1_exact > gpurun_out/r3_exact_sass.csv 2>&1
ncu -i gpurun_out/r3_v2_full.ncu-rep --page source --csv --print-source sass -k regex:k_s1_v2 > gpurun_out/r3_v2_sass.csv 2>&1
ls -la gpurun_out/r3*
