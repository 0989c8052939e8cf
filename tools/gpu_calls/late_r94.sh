mkdir -p gpurun_out
for c in B A E200; do python tools/s1_ab.py $c CURAST_LIB=tools/ab/base.so:CURAST_LIB=tools/ab/h2.so:CURAST_LIB=tools/ab/h2m7.so 10 2 >> gpurun_out/late94_ab.jsonl 2>&1; done
for l in base h2 h2m7; do for c in B A E200; do CURAST_LIB=tools/ab/$l.so python tools/ktimes.py $c 10 > gpurun_out/late94_kt_${l}_$c.json 2>&1; done; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -m gpu -p no:cacheprovider > gpurun_out/late94_tests.log 2>&1; echo "rc=$?" >> gpurun_out/late94_tests.log
