mkdir -p gpurun_out
for c in B E200; do python tools/s1_ab.py $c default:AB_CHUNK=1536:AB_CHUNK=1280:AB_CHUNK=1024:AB_CHUNK=1792 10 1 >> gpurun_out/late85_ab.jsonl 2>&1; done
