mkdir -p gpurun_out
rm -f gpurun_out/r18_ab.jsonl
for c in C A4 Bq; do python tools/s1_ab.py $c default 20 1 >> gpurun_out/r18_ab.jsonl 2>&1; done
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r18_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r18_tests.log
