mkdir -p gpurun_out
for e in 4 3 0; do CURAST_SPEC=$e python tools/ktimes.py B 2>/dev/null | grep "^{" >> gpurun_out/late41_kt.jsonl; done
python tools/s1_ab.py B default:CURAST_SPEC=0:CURAST_SPEC=3 20 2 > gpurun_out/late41_ab_B.jsonl 2>&1
