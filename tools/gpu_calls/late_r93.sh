mkdir -p gpurun_out
for l in base p6; do for c in A E200; do CURAST_LIB=tools/ab/$l.so python tools/ktimes.py $c 10 > gpurun_out/late93_kt_${l}_$c.json 2>&1; done; done
