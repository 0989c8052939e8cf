mkdir -p gpurun_out
for e in 4 3 0; do CURAST_SPEC=$e python tools/ktimes.py B 2>/dev/null | grep "^{" >> gpurun_out/late40_kt.jsonl; done
