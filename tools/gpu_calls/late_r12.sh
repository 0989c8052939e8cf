mkdir -p gpurun_out
for c in B C D; do
python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/pk.so+CURAST_F32_PACKED=1 15 2 > gpurun_out/r12_ab_$c.jsonl 2>&1
done
