mkdir -p gpurun_out
python tools/bimodal_procs.py 10 20 > gpurun_out/r27_procs.jsonl 2>&1
