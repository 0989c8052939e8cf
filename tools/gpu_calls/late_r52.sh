mkdir -p gpurun_out
for c in A B D E200; do python tools/s1_ab.py $c AB_ROW_RASTER=0:AB_ROW_RASTER=1 10 2 >> gpurun_out/late52_ab.jsonl 2>&1; done
