mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_H2=4:CURAST_H2=5:CURAST_H2=6 15 2 > gpurun_out/late63_ab.jsonl 2>&1
python tools/s1_ab.py E200 default:CURAST_H2=5:CURAST_H2=6 10 1 >> gpurun_out/late63_ab.jsonl 2>&1
python tools/s1_ab.py C default:CURAST_H2=5:CURAST_H2=6 10 1 >> gpurun_out/late63_ab.jsonl 2>&1
