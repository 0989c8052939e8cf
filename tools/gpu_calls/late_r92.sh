mkdir -p gpurun_out
for c in B A E200; do python tools/s1_ab.py $c CURAST_LIB=tools/ab/base.so:CURAST_LIB=tools/ab/p4.so:CURAST_LIB=tools/ab/p5.so:CURAST_LIB=tools/ab/p6.so:CURAST_LIB=tools/ab/p4i4.so 10 2 >> gpurun_out/late92_ab.jsonl 2>&1; done
for l in base p4 p5 p6 p4i4; do CURAST_LIB=tools/ab/$l.so python tools/ktimes.py B 10 > gpurun_out/late92_kt_${l}_B.json 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -m gpu -p no:cacheprovider > gpurun_out/late92_tests.log 2>&1; echo "rc=$?" >> gpurun_out/late92_tests.log
