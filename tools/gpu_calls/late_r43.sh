mkdir -p gpurun_out
python tools/phase_trace.py 3000 > gpurun_out/late43_trace.jsonl 2>&1
