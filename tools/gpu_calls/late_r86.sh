mkdir -p gpurun_out
python tools/s1_ab.py B default:AB_CHUNK=1792:AB_CHUNK=1920:AB_CHUNK=1664 10 2 >> gpurun_out/late86_ab.jsonl 2>&1
python tools/s1_ab.py Bq default:AB_CHUNK=1792 10 1 >> gpurun_out/late86_ab.jsonl 2>&1
python tools/s1_ab.py E200 default:AB_CHUNK=1792:AB_CHUNK=1536 8 1 >> gpurun_out/late86_ab.jsonl 2>&1
