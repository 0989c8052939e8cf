mkdir -p gpurun_out
for c in B A; do python tools/s1_ab.py $c CURAST_LIB=tools/ab/base.so:CURAST_LIB=tools/ab/ilp2.so:CURAST_LIB=tools/ab/ilp4m6.so 10 2 >> gpurun_out/late91_ab.jsonl 2>&1; done
for l in base ilp2 ilp4m6; do for c in B A; do CURAST_LIB=tools/ab/$l.so python tools/ktimes.py $c 10 > gpurun_out/late91_kt_${l}_$c.json 2>&1; done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "quad_pair" > gpurun_out/late91_tests.log 2>&1; echo "rc=$?" >> gpurun_out/late91_tests.log
