mkdir -p gpurun_out
python tools/bimodal.py 10 15 B > gpurun_out/r19_bimodal_1.jsonl 2>&1
python tools/bimodal.py 10 15 B > gpurun_out/r19_bimodal_2.jsonl 2>&1
