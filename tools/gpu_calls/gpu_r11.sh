mkdir -p gpurun_out
for c in A B C D Bq Dq; do python tools/s1_ab.py $c default 20 1 >> gpurun_out/r11_ab.jsonl 2>&1; done
python tools/s1_ab.py D CURAST_INSTANCED_KERNEL=0 10 1 >> gpurun_out/r11_ab.jsonl 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r11_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r11_tests.log
