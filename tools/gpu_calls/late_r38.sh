mkdir -p gpurun_out
for c in D Bq Dq C A; do python tools/ktimes.py $c 5 2>/dev/null | grep "^{" >> gpurun_out/late38_kt.jsonl; done
