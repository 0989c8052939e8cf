mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_LIB=tools/ab/base.so 20 3 > gpurun_out/late90_ab.jsonl 2>&1
for c in E200 C A D; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/base.so 10 2 >> gpurun_out/late90_ab.jsonl 2>&1; done
timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/late90_tests.log 2>&1; echo "rc=$?" >> gpurun_out/late90_tests.log
