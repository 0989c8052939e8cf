mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_LIB=tools/ab/base.so 20 3 > gpurun_out/late96_ab.jsonl 2>&1
for c in C A E200 Bq A4; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/base.so 10 2 >> gpurun_out/late96_ab.jsonl 2>&1; done
for l in default base; do if [ $l = base ]; then export CURAST_LIB=tools/ab/base.so; fi; python tools/ktimes.py B 10 > gpurun_out/late96_kt_${l}_B.json 2>&1; done; unset CURAST_LIB
timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/late96_tests.log 2>&1; echo "rc=$?" >> gpurun_out/late96_tests.log
